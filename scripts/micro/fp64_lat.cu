// Microbenchmark: dependent-chain latency of FP64 / FP32 / INT / LDS ops and FP64 throughput
// on the GPU box (developer tool). nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, double a, float fa, int ia) {
    __shared__ double sm[256];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double x = a; float y = fa; int z = ia;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) x = x + 1e-9; }  // DADD chain
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) x = x * 1.0000001; }  // DMUL chain
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) x = fma(x, 1.0000001, 1e-9); }  // DFMA chain
    long long t3 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) y = y * 1.0001f + 1e-5f; }  // FFMA chain
    long long t4 = clock64();
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) z = z * 3 + 1; }  // IMAD chain
    long long t5 = clock64();
    int k = threadIdx.x & 255;
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) k = ((int)sm[k] + 1) & 255; }  // LDS chain (+ F2I)
    long long t6 = clock64();
    bool p = x > 0;
#pragma unroll 1
    for (int i = 0; i < 100; ++i) {
#pragma unroll
 for (int j = 0; j < 10; ++j) { x = (x > 1.5) ? x - 0.5 : x + 0.25; } }  // DSETP+select+DADD chain
    long long t7 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
    }
    out[threadIdx.x] = x + y + z + k + p;
}
__global__ void thr(double *out, double a, int n) {  // independent DFMA streams: throughput
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, 1.0000001, 1e-9); x1 = fma(x1, 1.0000001, 1e-9); x2 = fma(x2, 1.0000001, 1e-9); x3 = fma(x3, 1.0000001, 1e-9);
        x4 = fma(x4, 1.0000001, 1e-9); x5 = fma(x5, 1.0000001, 1e-9); x6 = fma(x6, 1.0000001, 1e-9); x7 = fma(x7, 1.0000001, 1e-9);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 1 << 26); cudaMallocManaged(&c, 64);
    lat<<<1, 32>>>(o, c, 1.0, 1.0f, 1); cudaDeviceSynchronize();
    lat<<<1, 32>>>(o, c, 1.0, 1.0f, 1); cudaDeviceSynchronize();
    const char *nm[] = {"DADD", "DMUL", "DFMA", "FFMA", "IMAD", "LDS+cvt", "DSETP+FSEL+DADD"};
    for (int i = 0; i < 7; ++i) printf("%-8s %.1f cycles/op (dependent)\n", nm[i], c[i] / 1000.0);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int n = 4096, blocks = sms * 8, threads = 256;
    thr<<<blocks, threads>>>(o, 1.0, n); cudaDeviceSynchronize();
    cudaEventRecord(e0); thr<<<blocks, threads>>>(o, 1.0, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * n * 8;
    printf("DFMA throughput: %.2f TFMA/s = %.1f FMA/clk/SM at 1.965 GHz\n", fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}
