// Roofline denominators measured on the device the path runs on (bench.py reports the
// headline kernels against them; "measure the L2 gather peak on the box
// with an L2-resident gather microbenchmark, because NVIDIA does not publish it").
//
//   cs_bench_gather(mode, bytes, ...)  random 32-byte-sector gathers from an L2-resident
//       buffer of `bytes`, every SM busy; returns the achieved sector bandwidth (GB/s).
//       mode 0: ld.global.cg (L2 only: the L2 gather peak)
//       mode 1: ld.global.nc (__ldg: L1 + L2, the plain-global path of the kernels)
//       mode 2: tld4 on a 2D layered float texture (the texture path of sample_axes;
//               16 bytes of texels per fetch)
//       mode 3: streaming 16-byte loads over a buffer far above L2 (the HBM read peak)
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/contactsim_b200.h"
#include "cs_common.cuh"

namespace cs {
namespace {

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

constexpr int ROUNDS = 64;

template <int MODE>
__global__ void __launch_bounds__(256) k_gather(const float4 *__restrict__ buf, uint32_t n_sectors, float *sink,
                                                unsigned long long tex, int tw, int th, int tl) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.0f;
    uint32_t h = mix(tid * 2654435761u + 12345u);
#pragma unroll 8
    for (int r = 0; r < ROUNDS; ++r) {
        h = mix(h + (uint32_t)r);
        if (MODE == 2) {
            const int x = (int)(h % (uint32_t)(tw - 1)), y = (int)((h >> 8) % (uint32_t)(th - 1)),
                      l = (int)((h >> 20) % (uint32_t)tl);
            const float4 q = gather_a2d(tex, l, (float)(x + 1), (float)(y + 1));
            acc += q.x + q.y + q.z + q.w;
        } else {
            const uint32_t s = h % n_sectors;
            float4 v;
            if (MODE == 0) v = __ldcg(buf + 2 * (size_t)s);
            else v = __ldg(buf + 2 * (size_t)s);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1.2345f) sink[tid] = acc;  // never true in practice: keeps the loads
}

__global__ void __launch_bounds__(256) k_stream(const float4 *__restrict__ buf, size_t n, float *sink) {
    float acc = 0.0f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldcs(buf + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

}  // namespace
}  // namespace cs

using namespace cs;

extern "C" int cs_bench_gather(int32_t mode, int64_t bytes, int32_t iters, double *gbs) {
    if (!gbs || bytes < (1 << 20) || iters < 1 || mode < 0 || mode > 3) return CS_ERR_VALUE;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return CS_ERR_CUDA;
    float4 *buf = nullptr;
    float *sink = nullptr;
    cudaArray_t arr = nullptr;
    cudaTextureObject_t tex = 0;
    int tw = 0, th = 0, tl = 0;
    cudaEvent_t a = nullptr, b = nullptr;
    int rc = CS_OK;
    const size_t threads = (size_t)sms * 32 * 256;  // 32 CTAs of 256 per SM: every SM full
    do {
        if (cudaMalloc(&buf, (size_t)bytes) != cudaSuccess || cudaMalloc(&sink, threads * sizeof(float)) != cudaSuccess) {
            rc = CS_ERR_OOM;
            break;
        }
        cudaMemset(buf, 0, (size_t)bytes);
        if (mode == 2) {  // a layered texture of about `bytes`: 512 x 512 texels per layer
            tw = 512; th = 512; tl = (int)(bytes / (512 * 512 * 4));
            if (tl < 1) tl = 1;
            if (tl > 2048) tl = 2048;
            cudaChannelFormatDesc cf = cudaCreateChannelDesc<float>();
            if (cudaMalloc3DArray(&arr, &cf, make_cudaExtent(tw, th, tl), cudaArrayLayered) != cudaSuccess) { rc = CS_ERR_OOM; break; }
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeArray;
            rd.res.array.array = arr;
            cudaTextureDesc td{};
            td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
            td.filterMode = cudaFilterModePoint;
            td.readMode = cudaReadModeElementType;
            if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) { rc = CS_ERR_CUDA; break; }
        }
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const uint32_t nsec = (uint32_t)(bytes / 32);
        const unsigned grid = (unsigned)(threads / 256);
        auto launch = [&]() {
            switch (mode) {
                case 0: k_gather<0><<<grid, 256>>>(buf, nsec, sink, 0, 0, 0, 0); break;
                case 1: k_gather<1><<<grid, 256>>>(buf, nsec, sink, 0, 0, 0, 0); break;
                case 2: k_gather<2><<<grid, 256>>>(buf, nsec, sink, (unsigned long long)tex, tw, th, tl); break;
                default: k_stream<<<(unsigned)sms * 8, 256>>>(buf, (size_t)bytes / 16, sink); break;
            }
        };
        launch();  // warm: the buffer comes into L2 (modes 0-2)
        launch();
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(b);
        if (cudaEventSynchronize(b) != cudaSuccess) { rc = CS_ERR_CUDA; break; }
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        const double per = mode == 3 ? (double)bytes : (double)threads * ROUNDS * (mode == 2 ? 16.0 : 32.0);
        *gbs = per * iters / (ms * 1e-3) / 1e9;
    } while (0);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    if (tex) cudaDestroyTextureObject(tex);
    if (arr) cudaFreeArray(arr);
    cudaFree(buf);
    cudaFree(sink);
    if (rc == CS_OK && cudaGetLastError() != cudaSuccess) rc = CS_ERR_CUDA;
    return rc;
}
