// extern "C" boundary of libcontactsim_b200.so (include/contactsim_b200.h).
// Host-side state: SDF / mesh handle tables (fixed-capacity device descriptor
// arrays, so captured CUDA graphs stay valid across registrations), plans, and
// the thread-local error string the Python shim turns into the reference's
// exception classes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "cs_reduce.cuh"
#include "cs_sdfgen.cuh"
#include "cs_solver.cuh"
#include "cs_broadphase.cuh"

using namespace cs;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CS_CUDA(call)                                                                                    \
    do {                                                                                                 \
        cudaError_t _e = (call);                                                                         \
        if (_e != cudaSuccess)                                                                           \
            return fail(_e == cudaErrorMemoryAllocation ? CS_ERR_OOM : CS_ERR_CUDA, "%s: %s (%s:%d)", #call, \
                        cudaGetErrorString(_e), __FILE__, __LINE__);                                     \
    } while (0)

#define CS_LAUNCHED()                                                                                      \
    do {                                                                                                   \
        cudaError_t _e = cudaGetLastError();                                                               \
        if (_e != cudaSuccess) return fail(CS_ERR_CUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(_e), \
                                           __FILE__, __LINE__);                                            \
    } while (0)

constexpr int MAX_HANDLES = 4096;

struct SdfEntry {
    bool live = false;
    float *values = nullptr;
    float *cwin = nullptr;  // cell-window minima (GridT::cwin)
    float *bwin = nullptr;  // brick-window minima (GridT::bwin)
    cudaArray_t arr = nullptr;       // the values as a 2D layered texture (GridT::tex)
    cudaTextureObject_t tex = 0;
    size_t bytes = 0;
    SdfDesc desc{};
    int users = 0;        // live plans naming this grid
    bool doomed = false;  // freed by the caller while in use: released with the last plan
};
struct MeshEntry {
    bool live = false;
    double4 *verts = nullptr;
    int4 *tris = nullptr;
    int32_t *chunk_voff = nullptr, *chunk_verts = nullptr;
    uint2 *face_loc = nullptr;
    MeshDesc desc{};
    std::vector<int32_t> chunk_voff_h;  // host copy (k_face_prep block map)
    int users = 0;
    bool doomed = false;
};

std::mutex g_mu;
std::vector<SdfEntry> g_sdf;
std::vector<MeshEntry> g_mesh;
SdfDesc *d_sdfs = nullptr;
MeshDesc *d_meshes = nullptr;
int g_sms = 0;

int ensure_tables() {
    if (d_sdfs) return CS_OK;
    CS_CUDA(cudaMalloc(&d_sdfs, sizeof(SdfDesc) * MAX_HANDLES));
    CS_CUDA(cudaMalloc(&d_meshes, sizeof(MeshDesc) * MAX_HANDLES));
    CS_CUDA(cudaMemset(d_sdfs, 0, sizeof(SdfDesc) * MAX_HANDLES));
    CS_CUDA(cudaMemset(d_meshes, 0, sizeof(MeshDesc) * MAX_HANDLES));
    int dev = 0;
    CS_CUDA(cudaGetDevice(&dev));
    CS_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
    g_sdf.resize(MAX_HANDLES);
    g_mesh.resize(MAX_HANDLES);
    return CS_OK;
}

bool finite3(const double *v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

template <class T>
int dalloc(T **p, size_t n) {
    *p = nullptr;
    if (n == 0) n = 1;
    CS_CUDA(cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T)));
    return CS_OK;
}

// (g_mu held) device memory of a store entry
int free_sdf_entry(SdfEntry &s) {
    CS_CUDA(cudaFree(s.values));
    CS_CUDA(cudaFree(s.cwin));
    CS_CUDA(cudaFree(s.bwin));
    if (s.tex) CS_CUDA(cudaDestroyTextureObject(s.tex));
    if (s.arr) CS_CUDA(cudaFreeArray(s.arr));
    s = SdfEntry{};
    return CS_OK;
}
int free_mesh_entry(MeshEntry &m) {
    CS_CUDA(cudaFree(m.verts));
    CS_CUDA(cudaFree(m.tris));
    CS_CUDA(cudaFree(m.chunk_voff));
    CS_CUDA(cudaFree(m.chunk_verts));
    CS_CUDA(cudaFree(m.face_loc));
    m = MeshEntry{};
    return CS_OK;
}
// a plan stops using its assets: entries freed by the caller meanwhile go now
void release_assets(const std::vector<int32_t> &sdfs, const std::vector<int32_t> &meshes) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int32_t h : sdfs)
        if (--g_sdf[h].users == 0 && g_sdf[h].doomed) free_sdf_entry(g_sdf[h]);
    for (int32_t h : meshes)
        if (--g_mesh[h].users == 0 && g_mesh[h].doomed) free_mesh_entry(g_mesh[h]);
}

}  // namespace

struct cs_plan {
    int64_t E = 0;
    int32_t stages = 0;
    ReduceParams rp{};
    int64_t max_batch = 1;
    int64_t total_cap = 0;
    unsigned char *row_arena = nullptr;  // per-row buffers of the descent and of the reduction (aliased)
    int64_t nblocks = 0;
    bool uniform_sdf = false;      // every env samples the same grid
    PlanGrid uniform_grid{};  // ...whose view then travels as a kernel parameter
    bool uniform_mesh = false;     // every env uses the same mesh
    MeshDesc uniform_mesh_desc{};  // ...whose descriptor travels as a kernel parameter
    std::vector<void *> allocs;
    int64_t device_bytes = 0;
    // inputs / tables
    int32_t *env_sdf = nullptr, *env_mesh = nullptr;
    int64_t *cand_base = nullptr;
    int2 *block_map = nullptr;       // k_face_prep block -> (env, first face of the chunk)
    int4 *prep_map = nullptr;        // ... and (env, first face, chunk vertex offset, vertex count | mesh << 16)
    int32_t *chunk_first = nullptr;  // [E+1] first k_face_prep block of each env
    int32_t max_chunk_verts = 1;     // largest chunk vertex list over the plan's meshes
    EnvXf *xf = nullptr;
    Staging st{};
    Candidates cands{};
    ReduceIO io{};
    cs_outputs out{};
    // host e2e staging
    double *in_sdf = nullptr, *in_mesh = nullptr, *in_cd = nullptr;
    // cs_collide_host replays the collide from a CUDA graph captured on its second call
    // (the first, eager, does the lazy setup); none while phase timing is on
    cudaGraphExec_t host_exec = nullptr;
    cudaStream_t host_cap = nullptr;
    int32_t host_fmt = -1, host_calls = 0;
    bool host_graph_failed = false;
    int32_t *status = nullptr;
    double *env_min_depth = nullptr;  // scene semantics: min_depth None -> -cd per env
    unsigned long long *sample_counter = nullptr;  // non-null: counting builds ([0] prep, [1] pgd)
    unsigned long long *counter_buf = nullptr;
    // phase timing: ring of `timing_slots` steps x CS_TIMING_EVENTS events
    std::vector<cudaEvent_t> events;
    int64_t timing_step = 0;
    int32_t timing_slots = 0;
    // contact solver rows (cs_plan_solve / cs_multipair_solve), allocated on first use
    cs_solver_rows srows{}, mrows{};
    double *spacked = nullptr, *mpacked = nullptr;  // packed sweep records (launch_sweeps_packed)
    int32_t *mrow_count = nullptr;
    int64_t mrows_sys = 0;

    template <class T>
    int alloc(T **p, size_t n) {
        int r = dalloc(p, n);
        if (r == CS_OK) { allocs.push_back(*p); device_bytes += n * sizeof(T); }
        return r;
    }
    // assets this plan samples (their store entries outlive it, cs_sdf_free / cs_mesh_free)
    std::vector<int32_t> sdf_used, mesh_used;
    FinFork fork{};        // side streams of the finalize's concurrent branches (created lazily)
    bool fork_ready = false;
    const FinFork *get_fork() {
#ifdef CS_NO_FORK
        return nullptr;
#endif
        if (!fork_ready) {
            if (cudaStreamCreateWithFlags(&fork.s_block, cudaStreamNonBlocking) != cudaSuccess ||
                cudaStreamCreateWithFlags(&fork.s_fold, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&fork.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&fork.ev_block, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&fork.ev_fold, cudaEventDisableTiming) != cudaSuccess)
                return nullptr;  // no fork: the finalize runs in stream order
            fork_ready = true;
        }
        return &fork;
    }
    ~cs_plan() {
        if (host_exec) cudaGraphExecDestroy(host_exec);
        if (host_cap) cudaStreamDestroy(host_cap);
        if (fork_ready) {
            cudaStreamDestroy(fork.s_block); cudaStreamDestroy(fork.s_fold);
            cudaEventDestroy(fork.ev_fork); cudaEventDestroy(fork.ev_block); cudaEventDestroy(fork.ev_fold);
        }
        for (cudaEvent_t e : events) cudaEventDestroy(e);
        for (void *p : allocs) cudaFree(p);
        release_assets(sdf_used, mesh_used);
    }
};

extern "C" {

const char *cs_last_error(void) { return g_err.c_str(); }

int cs_abi_version(void) { return CS_ABI_VERSION; }

int cs_device_info(int32_t *sm_count, int64_t *l2_bytes, int64_t *persist_l2_max) {
    int dev = 0, v = 0;
    CS_CUDA(cudaGetDevice(&dev));
    CS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    if (sm_count) *sm_count = v;
    CS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev));
    if (l2_bytes) *l2_bytes = v;
    CS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev));
    if (persist_l2_max) *persist_l2_max = v;
    return CS_OK;
}

// ---------------------------------------------------------------- SDF store

static int check_grid_args(int32_t nx, int32_t ny, int32_t nz, double voxel) {
    if (nx < 2 || ny < 2 || nz < 2) return fail(CS_ERR_VALUE, "grid dims must be at least 2 per axis");
    if (!(voxel > 0.0)) return fail(CS_ERR_VALUE, "voxel_size must be positive");
    const int64_t n = (int64_t)nx * ny * nz;
    if (n >= (int64_t)1 << 31) return fail(CS_ERR_VALUE, "grid of %lld voxels exceeds the 2^31 device index range", (long long)n);
    return CS_OK;
}

// A free SDF slot (g_mu held); -1 when the table is full.
static int free_sdf_slot() {
    for (int i = 0; i < MAX_HANDLES; ++i)
        if (!g_sdf[i].live) return i;
    return -1;
}

static int finish_sdf_register(int h, int32_t nx, int32_t ny, int32_t nz, const double origin[3], double voxel,
                               const double aabb_lo[3], const double aabb_hi[3], int32_t *handle);

int cs_sdf_register(const float *values, int values_on_device, int32_t nx, int32_t ny, int32_t nz,
                    const double origin[3], double voxel, const double aabb_lo[3], const double aabb_hi[3],
                    int32_t *handle) {
    int r = check_grid_args(nx, ny, nz, voxel);
    if (r) return r;
    const int64_t n = (int64_t)nx * ny * nz;
    if (!values || !handle || !origin || !aabb_lo || !aabb_hi) return fail(CS_ERR_VALUE, "null argument");
    std::lock_guard<std::mutex> lk(g_mu);
    r = ensure_tables();
    if (r) return r;
    const int h = free_sdf_slot();
    if (h < 0) return fail(CS_ERR_HANDLE, "SDF handle table full (%d)", MAX_HANDLES);
    SdfEntry &s = g_sdf[h];
    s.bytes = (size_t)n * sizeof(float);
    CS_CUDA(cudaMalloc(&s.values, s.bytes));
    CS_CUDA(cudaMemcpy(s.values, values, s.bytes, values_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    return finish_sdf_register(h, nx, ny, nz, origin, voxel, aabb_lo, aabb_hi, handle);
}

// The CSIMSDF1 file (sdf/grid.py:138-160: "<8s3i d 3d 6d" header, then float32
// values) straight into the device store: the values stream from the file through two
// pinned staging buffers (a read overlaps the previous chunk's copy), never as a host array.
int cs_sdf_register_file(const char *path, int32_t *handle, cs_sdf_file_info *info) {
    if (!path || !handle) return fail(CS_ERR_VALUE, "null argument");
    FILE *fh = std::fopen(path, "rb");
    if (!fh) return fail(CS_ERR_IO, "cannot open %s", path);
    unsigned char head[100];
    if (std::fread(head, 1, sizeof(head), fh) != sizeof(head)) { std::fclose(fh); return fail(CS_ERR_VALUE, "not an SDF grid file: %s", path); }
    if (std::memcmp(head, "CSIMSDF1", 8) != 0) { std::fclose(fh); return fail(CS_ERR_VALUE, "not an SDF grid file: %s", path); }
    int32_t dims[3];
    double voxel, origin[3], aabb[6];
    std::memcpy(dims, head + 8, 12);
    std::memcpy(&voxel, head + 20, 8);
    std::memcpy(origin, head + 28, 24);
    std::memcpy(aabb, head + 52, 48);
    int r = check_grid_args(dims[0], dims[1], dims[2], voxel);
    if (r) { std::fclose(fh); return r; }
    const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    std::lock_guard<std::mutex> lk(g_mu);
    r = ensure_tables();
    if (r) { std::fclose(fh); return r; }
    const int h = free_sdf_slot();
    if (h < 0) { std::fclose(fh); return fail(CS_ERR_HANDLE, "SDF handle table full (%d)", MAX_HANDLES); }
    SdfEntry &s = g_sdf[h];
    s.bytes = (size_t)n * sizeof(float);
    constexpr size_t CHUNK = (size_t)8 << 20;
    unsigned char *stage = nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&]() {
        if (stage) cudaFreeHost(stage);
        for (auto e : ev) if (e) cudaEventDestroy(e);
        if (cs) cudaStreamDestroy(cs);
        std::fclose(fh);
    };
    cudaError_t ce = cudaMalloc(&s.values, s.bytes);
    if (ce == cudaSuccess) ce = cudaHostAlloc(&stage, 2 * CHUNK, cudaHostAllocDefault);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    size_t done = 0;
    int k = 0;
    bool truncated = false;
    while (ce == cudaSuccess && done < s.bytes) {
        const size_t want = std::min(CHUNK, s.bytes - done);
        unsigned char *buf = stage + (size_t)k * CHUNK;
        ce = cudaEventSynchronize(ev[k]);  // the copy that last used this buffer is done
        if (ce != cudaSuccess) break;
        if (std::fread(buf, 1, want, fh) != want) { truncated = true; break; }
        ce = cudaMemcpyAsync(reinterpret_cast<unsigned char *>(s.values) + done, buf, want, cudaMemcpyHostToDevice, cs);
        if (ce == cudaSuccess) ce = cudaEventRecord(ev[k], cs);
        done += want;
        k ^= 1;
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(cs);
    cleanup();
    if (ce != cudaSuccess || truncated) {
        cudaFree(s.values);
        s.values = nullptr;
        if (truncated) return fail(CS_ERR_VALUE, "values length does not match dims: %s", path);
        return fail(CS_ERR_CUDA, "%s: %s", path, cudaGetErrorString(ce));
    }
    if (info) {
        for (int a = 0; a < 3; ++a) {
            info->dims[a] = dims[a];
            info->origin[a] = origin[a];
            info->aabb_lo[a] = aabb[a];
            info->aabb_hi[a] = aabb[3 + a];
        }
        info->voxel = voxel;
    }
    return finish_sdf_register(h, dims[0], dims[1], dims[2], origin, voxel, aabb, aabb + 3, handle);
}

// The device-side tables of a grid whose values are in g_sdf[h].values (g_mu held).
static int finish_sdf_register(int h, int32_t nx, int32_t ny, int32_t nz, const double origin[3], double voxel,
                               const double aabb_lo[3], const double aabb_hi[3], int32_t *handle) {
    SdfEntry &s = g_sdf[h];
    GridT<float> probe = cs::make_grid<float>(nullptr, nx, ny, nz, origin[0], origin[1], origin[2], voxel);
    // brick-window minima (the first pass of the face lower bound, cs_common.cuh:
    // sample_lower_bound), built on the device, and a scan of the values: non-finite
    // values disable the bound; the largest |value| sets its absolute rounding margin
    unsigned scan_h[2] = {0, 0};
    {
        const int bx = probe.bnx, by = probe.bny, bz = probe.bnz;
        const size_t nb = (size_t)bx * by * bz;
        float *bm = nullptr;
        unsigned *scan = nullptr;
        CS_CUDA(cudaMalloc(&s.bwin, 8 * nb * sizeof(float)));
        CS_CUDA(cudaMalloc(&bm, nb * sizeof(float)));
        CS_CUDA(cudaMalloc(&scan, 2 * sizeof(unsigned)));
        build_brick_windows(s.values, nx, ny, nz, bx, by, bz, bm, s.bwin, scan, 0);
        CS_CUDA(cudaGetLastError());
        CS_CUDA(cudaMemcpy(scan_h, scan, sizeof(scan_h), cudaMemcpyDeviceToHost));
        CS_CUDA(cudaFree(bm));
        CS_CUDA(cudaFree(scan));
    }
    {   // cell-window minima of the exact face bound (cs_common.cuh: sample_lower_bound)
        const int64_t nc = (int64_t)(nx - 1) * (ny - 1) * (nz - 1);
        float *tmp = nullptr;
        CS_CUDA(cudaMalloc(&s.cwin, (size_t)CWIN_LEVELS * nc * sizeof(float)));
        CS_CUDA(cudaMalloc(&tmp, (size_t)nc * sizeof(float)));
        build_cell_windows(s.values, nx, ny, nz, s.cwin, tmp, 0);
        CS_CUDA(cudaGetLastError());
        CS_CUDA(cudaDeviceSynchronize());
        CS_CUDA(cudaFree(tmp));
    }
#ifndef CS_NO_TEX
    {   // the values as a 2D layered texture (x, y, layer z): tld4 returns a cell face's
        // 2 x 2 corners in one fetch (cs_common.cuh: sample_axes)
        cudaChannelFormatDesc cf = cudaCreateChannelDesc<float>();
        CS_CUDA(cudaMalloc3DArray(&s.arr, &cf, make_cudaExtent(nx, ny, nz), cudaArrayLayered));
        cudaMemcpy3DParms cp{};
        cp.srcPtr = make_cudaPitchedPtr(s.values, (size_t)nx * sizeof(float), nx, ny);
        cp.dstArray = s.arr;
        cp.extent = make_cudaExtent(nx, ny, nz);
        cp.kind = cudaMemcpyDeviceToDevice;
        CS_CUDA(cudaMemcpy3D(&cp));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = s.arr;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CS_CUDA(cudaCreateTextureObject(&s.tex, &rd, &td, nullptr));
    }
#endif
    SdfDesc &d = s.desc;
    d.values = s.values;
    d.nx = nx; d.ny = ny; d.nz = nz; d.pad = 0;
    d.ox = origin[0]; d.oy = origin[1]; d.oz = origin[2];
    d.voxel = voxel;
    for (int k = 0; k < 3; ++k) { d.lo[k] = aabb_lo[k]; d.hi[k] = aabb_hi[k]; }
    d.gp = cs::make_grid<float>(s.values, nx, ny, nz, origin[0], origin[1], origin[2], voxel);
    d.gp.cwin = s.cwin;
    d.gp.bwin = s.bwin;
    if (scan_h[0]) {  // NaN / inf values: no bound (fminf would skip a NaN corner)
        d.gp.cwin = nullptr;
        d.gp.bwin = nullptr;
    }
    {
        float vmax;
        std::memcpy(&vmax, &scan_h[1], sizeof(float));
        d.gp.lbm = (double)vmax * 0x1p-40;  // see sample_lower_bound
    }
    d.gp.tex = 0;  // the texture is used by uniform-grid plans only (a warp-uniform handle: cs_plan_create)
    CS_CUDA(cudaMemcpy(d_sdfs + h, &d, sizeof(SdfDesc), cudaMemcpyHostToDevice));
    s.live = true;
    *handle = h;
    return CS_OK;
}

int cs_sdf_free(int32_t handle) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (handle < 0 || handle >= (int)g_sdf.size() || !g_sdf[handle].live || g_sdf[handle].doomed)
        return fail(CS_ERR_HANDLE, "bad SDF handle %d", handle);
    SdfEntry &s = g_sdf[handle];
    if (s.users > 0) {  // a live plan samples it: freed when the last such plan is destroyed
        s.doomed = true;
        return CS_OK;
    }
    return free_sdf_entry(s);
}

int cs_sdf_values(int32_t handle, const float **values) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (handle < 0 || handle >= (int)g_sdf.size() || !g_sdf[handle].live) return fail(CS_ERR_HANDLE, "bad SDF handle %d", handle);
    *values = g_sdf[handle].values;
    return CS_OK;
}

int cs_sdf_l2_persist(int32_t handle, void *stream, float hit_ratio) {
    void *base;
    size_t bytes;
    {   // the plan kernels gather from the float32 values: that is the array to keep resident
        std::lock_guard<std::mutex> lk(g_mu);
        if (handle < 0 || handle >= (int)g_sdf.size() || !g_sdf[handle].live) return fail(CS_ERR_HANDLE, "bad SDF handle %d", handle);
        base = g_sdf[handle].values;
        bytes = g_sdf[handle].bytes;
    }
    int dev = 0, max_win = 0, max_persist = 0;
    CS_CUDA(cudaGetDevice(&dev));
    CS_CUDA(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev));
    CS_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
    cudaStreamAttrValue attr;
    memset(&attr, 0, sizeof(attr));
    if (hit_ratio > 0.0f && max_win > 0 && max_persist > 0) {
        size_t win = std::min(bytes, (size_t)max_win);
        size_t persist = std::min(win, (size_t)max_persist);
        CS_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
        attr.accessPolicyWindow.base_ptr = base;
        attr.accessPolicyWindow.num_bytes = win;
        attr.accessPolicyWindow.hitRatio = std::min(1.0f, hit_ratio * (float)persist / (float)win);
        attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
        attr.accessPolicyWindow.num_bytes = 0;
    }
    CS_CUDA(cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &attr));
    return CS_OK;
}

// ---------------------------------------------------------------- mesh store

int cs_mesh_register(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int32_t *handle) {
    if (!vertices || !triangles || !handle) return fail(CS_ERR_VALUE, "null argument");
    if (nv < 3 || nt < 1) return fail(CS_ERR_MESH, "mesh needs at least 3 vertices and 1 triangle");
    if (nt >= ((int64_t)1 << 29)) return fail(CS_ERR_MESH, "too many triangles (limit 2^29)");
    std::vector<double4> v4((size_t)nv);
    for (int64_t i = 0; i < nv; ++i) {
        const double *p = vertices + 3 * i;
        if (!finite3(p)) return fail(CS_ERR_MESH, "non-finite vertex coordinate");
        v4[(size_t)i] = make_double4(p[0], p[1], p[2], 0.0);
    }
    std::vector<int4> t4((size_t)nt);
    for (int64_t i = 0; i < nt; ++i) {
        const int32_t *t = triangles + 3 * i;
        for (int k = 0; k < 3; ++k)
            if (t[k] < 0 || t[k] >= nv) return fail(CS_ERR_MESH, "triangle index out of range (have %lld vertices)", (long long)nv);
        t4[(size_t)i] = make_int4(t[0], t[1], t[2], 0);
    }
    // chunk-local vertex lists (k_face_prep samples each distinct vertex of a chunk once)
    const int64_t nchunks = (nt + FACE_CHUNK - 1) / FACE_CHUNK;
    std::vector<int32_t> voff((size_t)nchunks + 1), cverts;
    std::vector<uint2> floc((size_t)nt);
    int32_t maxcv = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t f0 = c * FACE_CHUNK, f1 = std::min<int64_t>(nt, f0 + FACE_CHUNK);
        std::vector<int32_t> ids;
        ids.reserve((size_t)(3 * (f1 - f0)));
        for (int64_t f = f0; f < f1; ++f)
            for (int k = 0; k < 3; ++k) ids.push_back(triangles[3 * f + k]);
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        voff[(size_t)c] = (int32_t)cverts.size();
        for (int64_t f = f0; f < f1; ++f) {
            uint32_t loc[3];
            for (int k = 0; k < 3; ++k)
                loc[k] = (uint32_t)(std::lower_bound(ids.begin(), ids.end(), triangles[3 * f + k]) - ids.begin());
            floc[(size_t)f] = make_uint2(loc[0] | (loc[1] << 16), loc[2]);
        }
        cverts.insert(cverts.end(), ids.begin(), ids.end());
        maxcv = std::max<int32_t>(maxcv, (int32_t)ids.size());
    }
    voff[(size_t)nchunks] = (int32_t)cverts.size();
    std::lock_guard<std::mutex> lk(g_mu);
    int r = ensure_tables();
    if (r) return r;
    int h = -1;
    for (int i = 0; i < MAX_HANDLES; ++i)
        if (!g_mesh[i].live) { h = i; break; }
    if (h < 0) return fail(CS_ERR_HANDLE, "mesh handle table full (%d)", MAX_HANDLES);
    MeshEntry &m = g_mesh[h];
    CS_CUDA(cudaMalloc(&m.verts, sizeof(double4) * (size_t)nv));
    CS_CUDA(cudaMalloc(&m.tris, sizeof(int4) * (size_t)nt));
    CS_CUDA(cudaMemcpy(m.verts, v4.data(), sizeof(double4) * (size_t)nv, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(m.tris, t4.data(), sizeof(int4) * (size_t)nt, cudaMemcpyHostToDevice));
    CS_CUDA(cudaMalloc(&m.chunk_voff, sizeof(int32_t) * voff.size()));
    CS_CUDA(cudaMalloc(&m.chunk_verts, sizeof(int32_t) * std::max<size_t>(1, cverts.size())));
    CS_CUDA(cudaMalloc(&m.face_loc, sizeof(uint2) * floc.size()));
    CS_CUDA(cudaMemcpy(m.chunk_voff, voff.data(), sizeof(int32_t) * voff.size(), cudaMemcpyHostToDevice));
    m.chunk_voff_h.assign(voff.begin(), voff.end());
    CS_CUDA(cudaMemcpy(m.chunk_verts, cverts.data(), sizeof(int32_t) * cverts.size(), cudaMemcpyHostToDevice));
    CS_CUDA(cudaMemcpy(m.face_loc, floc.data(), sizeof(uint2) * floc.size(), cudaMemcpyHostToDevice));
    m.desc.verts = m.verts;
    m.desc.tris = m.tris;
    m.desc.chunk_voff = m.chunk_voff;
    m.desc.chunk_verts = m.chunk_verts;
    m.desc.face_loc = m.face_loc;
    m.desc.nv = nv;
    m.desc.nt = nt;
    m.desc.nchunks = (int32_t)nchunks;
    m.desc.max_chunk_verts = maxcv;
    CS_CUDA(cudaMemcpy(d_meshes + h, &m.desc, sizeof(MeshDesc), cudaMemcpyHostToDevice));
    m.live = true;
    *handle = h;
    return CS_OK;
}

int cs_mesh_free(int32_t handle) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (handle < 0 || handle >= (int)g_mesh.size() || !g_mesh[handle].live || g_mesh[handle].doomed)
        return fail(CS_ERR_HANDLE, "bad mesh handle %d", handle);
    MeshEntry &m = g_mesh[handle];
    if (m.users > 0) {
        m.doomed = true;
        return CS_OK;
    }
    return free_mesh_entry(m);
}

// ---------------------------------------------------------------- per-pair drop-ins

static int make_grid(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                     double voxel, GridView *g) {
    if (nx < 2 || ny < 2 || nz < 2) return fail(CS_ERR_VALUE, "grid dims must be at least 2 per axis");
    if (nx * ny * nz >= ((int64_t)1 << 31)) return fail(CS_ERR_VALUE, "grid exceeds the 2^31 device index range");
    if (!(voxel > 0.0)) return fail(CS_ERR_VALUE, "voxel_size must be positive");
    *g = cs::make_grid<float>(values, (int)nx, (int)ny, (int)nz, ox, oy, oz, voxel);
    return CS_OK;
}

int cs_face_contacts(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                     double voxel, const double *tri_verts, int64_t m, double contact_distance, int32_t max_iters,
                     double tol, double *out_point, double *out_phi, double *out_grad, uint8_t *out_found,
                     void *stream) {
    GridView g;
    int r = make_grid(values, nx, ny, nz, ox, oy, oz, voxel, &g);
    if (r) return r;
    if (m < 0) return fail(CS_ERR_VALUE, "negative face count");
    launch_face_contacts(g, tri_verts, m, contact_distance, max_iters, tol, out_point, out_phi, out_grad, out_found,
                         (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_sdf_sample(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                  double voxel, const double *points, int64_t n, double *out, void *stream) {
    GridView g;
    int r = make_grid(values, nx, ny, nz, ox, oy, oz, voxel, &g);
    if (r) return r;
    launch_sdf_sample(g, points, n, out, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_sdf_gradient(const float *values, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                    double voxel, const double *points, int64_t n, double *out, void *stream) {
    GridView g;
    int r = make_grid(values, nx, ny, nz, ox, oy, oz, voxel, &g);
    if (r) return r;
    launch_sdf_gradient(g, points, n, out, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

// ---------------------------------------------------------------- plans

static int check_params(const cs_reduction_params *p) {
    if (!p) return fail(CS_ERR_VALUE, "null ReductionParams");
    // contacts/types.py:70-78
    if (p->max_patches < 1) return fail(CS_ERR_VALUE, "max_patches must be positive");
    if (p->per_patch_cap < 1) return fail(CS_ERR_VALUE, "per_patch_cap must be at least 1");
    if (!(p->normal_cone_cos >= -1.0 && p->normal_cone_cos <= 1.0)) return fail(CS_ERR_VALUE, "normal_cone_cos must be a cosine");
    if (p->batch_size < 1) return fail(CS_ERR_VALUE, "batch_size must be positive");
    if (p->per_patch_cap > MAX_KEPT) return fail(CS_ERR_VALUE, "per_patch_cap above the GPU limit of %d", MAX_KEPT);
    if (p->max_patches > 4096) return fail(CS_ERR_VALUE, "max_patches above the GPU limit of 4096");
    return CS_OK;
}

static int plan_buffers(cs_plan *P, const std::vector<int64_t> &cap) {
    const int64_t E = P->E;
    std::vector<int64_t> base((size_t)E);
    int64_t tot = 0, maxcap = 1;
    for (int64_t e = 0; e < E; ++e) {
        base[(size_t)e] = tot;
        tot += cap[(size_t)e];
        maxcap = std::max(maxcap, cap[(size_t)e]);
    }
    if (tot >= ((int64_t)1 << 31)) return fail(CS_ERR_VALUE, "plan of %lld face rows exceeds the 2^31 row index range", (long long)tot);
    P->total_cap = tot;
    const int N = P->rp.N, K = P->rp.K;
    int r;
#define A(ptr, n) if ((r = P->alloc(&(ptr), (size_t)(n)))) return r
    A(P->cand_base, E);
    CS_CUDA(cudaMemcpy(P->cand_base, base.data(), sizeof(int64_t) * (size_t)E, cudaMemcpyHostToDevice));
    A(P->status, E);
    A(P->io.n_cand, E);
    A(P->cands.point, 3 * tot); A(P->cands.normal, 3 * tot); A(P->cands.depth, tot); A(P->cands.face, tot);
    // The descent's per-row staging is dead once k_compact has written the candidates,
    // and the reduction's per-row scratch is live only after it (both stream-ordered
    // within one collide; neither carries state across calls): one arena holds either.
    {
        const bool red = (P->stages & CS_STAGE_REDUCE) != 0;
        auto carve = [&](uintptr_t base, bool gen_side) {
            uintptr_t off = 0;
            auto take = [&](auto *&ptr, size_t n) {
                off = (off + 255) & ~(uintptr_t)255;
                ptr = reinterpret_cast<std::remove_reference_t<decltype(ptr)>>(base + off);
                off += n * sizeof(*ptr);
            };
            const size_t t = (size_t)tot;
            if (gen_side) {
                Staging &st = P->st;
                take(st.point, 3 * t); take(st.phi, t); take(st.grad, 3 * t); take(st.face, t); take(st.work, t);
                take(st.alpha, t); take(st.acc, t); take(st.acc_hd, t); take(st.slow, t);
            } else {
                ReduceIO &q = P->io;
                take(q.order, t); take(q.label, t); take(q.su, t); take(q.sv, t); take(q.sp, t); take(q.suv, t);
                take(q.tuv, t); take(q.tpos, t); take(q.tu, t); take(q.tv, t); take(q.tk, t); take(q.fw, t); take(q.hj, 4 * t);
                take(q.hu, 4 * t); take(q.hv, 4 * t);
            }
            return (size_t)off;
        };
        const size_t gen_bytes = carve(0, true), red_bytes = red ? carve(0, false) : 0;
        A(P->row_arena, std::max(gen_bytes, red_bytes));
        carve(reinterpret_cast<uintptr_t>(P->row_arena), true);
        if (red) carve(reinterpret_cast<uintptr_t>(P->row_arena), false);
    }
    CS_CUDA(cudaMemset(P->status, 0, sizeof(int32_t) * (size_t)E));
    CS_CUDA(cudaMemset(P->io.n_cand, 0, sizeof(int32_t) * (size_t)E));
    ReduceIO &io = P->io;
    io.E = E;
    io.cand_base = P->cand_base;
    io.point = P->cands.point; io.normal = P->cands.normal; io.depth = P->cands.depth; io.face = P->cands.face;
    if (P->stages & CS_STAGE_REDUCE) {
        A(io.sh, 2 * tot + E * (4 * (int64_t)N + 4));
        A(io.hlen, 4 * E * N); A(io.pdeep, E * N); A(io.pnt, E * N); A(io.wenv, E * N);
        A(io.jobs, 64 * 4 * E * N); A(io.njob, 65);
        A(io.patch_off, E + 1); A(io.red_slow, E);
        A(io.large_list, E * N); A(io.large_count, 1);
        A(io.n_patch, E); A(io.n_kept, E);
        A(io.patch_normal, 3 * E * N); A(io.builder_maxd, E * N);
        A(io.member_offsets, E * (N + 1)); A(io.members, tot);
        A(io.patch_nkept, E * N); A(io.kept_cand, E * N * K); A(io.kept_face, E * N * K);
        A(io.kept_point, 3 * E * N * K); A(io.kept_normal, 3 * E * N * K); A(io.kept_depth, E * N * K);
        A(io.w_sum, E * N); A(io.wp_sum, 3 * E * N); A(io.wn_sum, 3 * E * N); A(io.wt_sum, 3 * E * N);
        A(io.area, E * N); A(io.max_depth, E * N);
        A(io.stats, 4 * E);
        CS_CUDA(cudaMemset(io.n_patch, 0, sizeof(int32_t) * (size_t)E));
        CS_CUDA(cudaMemset(io.stats, 0, sizeof(float) * 4 * (size_t)E));
    }
#undef A
    P->max_batch = std::min<int64_t>(P->rp.batch_size, maxcap);
    if (P->stages & CS_STAGE_REDUCE) {
        // k_reduce stages one batch and the builders in shared memory: refuse plans whose
        // (max_patches, batch_size) need more than the device's opt-in limit per block
        int dev = 0, optin = 0;
        CS_CUDA(cudaGetDevice(&dev));
        CS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        const size_t need = reduce_smem_bytes(N, (int)P->max_batch);
        if (need > (size_t)optin)
            return fail(CS_ERR_VALUE, "max_patches %d with batch_size %lld needs %zu bytes of shared memory per env "
                        "(device limit %d): lower batch_size or max_patches", N, (long long)P->max_batch, need, optin);
    }
    cs_outputs &o = P->out;
    o.n_envs = E;
    o.max_patches = N;
    o.per_patch_cap = K;
    o.total_capacity = tot;
    o.cand_base = P->cand_base;
    o.env_status = P->status;
    o.n_cand = io.n_cand;
    o.n_patch = io.n_patch; o.n_kept = io.n_kept; o.stats = io.stats;
    o.cand_point = P->cands.point; o.cand_normal = P->cands.normal; o.cand_depth = P->cands.depth;
    o.cand_face = P->cands.face;
    o.patch_normal = io.patch_normal; o.patch_nkept = io.patch_nkept; o.kept_cand = io.kept_cand;
    o.kept_point = io.kept_point; o.kept_normal = io.kept_normal; o.kept_depth = io.kept_depth;
    o.kept_face = io.kept_face;
    o.w_sum = io.w_sum; o.wp_sum = io.wp_sum; o.wn_sum = io.wn_sum; o.wt_sum = io.wt_sum;
    o.area = io.area; o.max_depth = io.max_depth;
    o.member_offsets = io.member_offsets; o.members = io.members;
    return CS_OK;
}

int cs_plan_create(int64_t n_envs, const int32_t *sdf_handles, const int32_t *mesh_handles,
                   const cs_reduction_params *params, int32_t stages, cs_plan **plan) {
    if (!plan) return fail(CS_ERR_VALUE, "null plan pointer");
    *plan = nullptr;
    if (n_envs < 1) return fail(CS_ERR_VALUE, "n_envs must be positive");
    if (!(stages & CS_STAGE_GENERATE)) return fail(CS_ERR_VALUE, "cs_plan_create needs the generate stage");
    if (stages & CS_STAGE_REDUCE) {
        int r = check_params(params);
        if (r) return r;
    }
    std::vector<int64_t> cap((size_t)n_envs);
    std::vector<int2> bmap;
    std::vector<int4> pmap;
    std::vector<int32_t> chunk_first;
    bool uniform = true;
    PlanGrid ugrid{};
    int32_t maxcv = 1;
    std::vector<int32_t> used_s, used_m;
    bool umesh = false;
    MeshDesc umdesc{};
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int r = ensure_tables();
        if (r) return r;
        for (int64_t e = 0; e < n_envs; ++e) {
            uniform &= sdf_handles[e] == sdf_handles[0];
            int s = sdf_handles[e], m = mesh_handles[e];
            if (s < 0 || s >= MAX_HANDLES || !g_sdf[s].live || g_sdf[s].doomed)
                return fail(CS_ERR_HANDLE, "env %lld: bad SDF handle %d", (long long)e, s);
            if (m < 0 || m >= MAX_HANDLES || !g_mesh[m].live || g_mesh[m].doomed)
                return fail(CS_ERR_HANDLE, "env %lld: bad mesh handle %d", (long long)e, m);
            int64_t nt = g_mesh[m].desc.nt;
            cap[(size_t)e] = nt;
            maxcv = std::max(maxcv, g_mesh[m].desc.max_chunk_verts);
            chunk_first.push_back((int32_t)bmap.size());
            const std::vector<int32_t> &vo = g_mesh[m].chunk_voff_h;
            for (int64_t f = 0; f < nt; f += FACE_CHUNK) {
                bmap.push_back(make_int2((int)e, (int)f));
                const int c = (int)(f / FACE_CHUNK);
                pmap.push_back(make_int4((int)e, (int)f, vo[c], (vo[c + 1] - vo[c]) | (m << 16)));
            }
        }
        if (uniform) {
            ugrid = g_sdf[sdf_handles[0]].desc.gp;
            // tld4 takes its texture handle in a uniform register: only plans whose envs
            // all sample one grid (the handle a kernel parameter) gather through it
            ugrid.tex = (unsigned long long)g_sdf[sdf_handles[0]].tex;
        }
        umesh = true;
        for (int64_t e = 0; e < n_envs; ++e) umesh &= mesh_handles[e] == mesh_handles[0];
        if (umesh) umdesc = g_mesh[mesh_handles[0]].desc;
        chunk_first.push_back((int32_t)bmap.size());
        used_s.assign(sdf_handles, sdf_handles + n_envs);
        used_m.assign(mesh_handles, mesh_handles + n_envs);
        for (auto *u : {&used_s, &used_m}) {
            std::sort(u->begin(), u->end());
            u->erase(std::unique(u->begin(), u->end()), u->end());
        }
        for (int32_t h : used_s) ++g_sdf[h].users;
        for (int32_t h : used_m) ++g_mesh[h].users;
    }
    cs_plan *P = new cs_plan();
    P->sdf_used = std::move(used_s);  // released by ~cs_plan (also on the failure paths below)
    P->mesh_used = std::move(used_m);
    P->E = n_envs;
    P->stages = stages;
    P->uniform_sdf = uniform;
    P->uniform_grid = ugrid;
    P->uniform_mesh = umesh;
    P->uniform_mesh_desc = umdesc;
    P->max_chunk_verts = maxcv;
    if (stages & CS_STAGE_REDUCE) {
        P->rp.N = params->max_patches; P->rp.K = params->per_patch_cap; P->rp.batch_size = params->batch_size;
        P->rp.has_min_depth = params->has_min_depth; P->rp.cone = params->normal_cone_cos; P->rp.min_depth = params->min_depth;
    } else {
        P->rp.N = 1; P->rp.K = 1; P->rp.batch_size = 1;
    }
    int r = plan_buffers(P, cap);
    if (!r) r = P->alloc(&P->env_sdf, (size_t)n_envs);
    if (!r) r = P->alloc(&P->env_mesh, (size_t)n_envs);
    if (!r) r = P->alloc(&P->block_map, bmap.size());
    if (!r) r = P->alloc(&P->prep_map, pmap.size());
    if (!r) r = P->alloc(&P->xf, (size_t)n_envs);
    if (!r) r = P->alloc(&P->st.chunk_count, bmap.size());
    if (!r) r = P->alloc(&P->st.chunk_off, bmap.size());
    if (!r) r = P->alloc(&P->st.chunk_found, bmap.size());
    if (!r) r = P->alloc(&P->st.work_count, 4);
    if (!r) r = P->alloc(&P->chunk_first, chunk_first.size());
    if (!r && (stages & CS_STAGE_REDUCE) && !params->has_min_depth) {
        r = P->alloc(&P->env_min_depth, (size_t)n_envs);
        P->io.env_min_depth = P->env_min_depth;
    }
    if (r) { delete P; return r; }
    P->nblocks = (int64_t)bmap.size();
    P->out.face_work = P->st.work_count;
    cudaError_t ce = cudaMemcpy(P->env_sdf, sdf_handles, sizeof(int32_t) * (size_t)n_envs, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(P->env_mesh, mesh_handles, sizeof(int32_t) * (size_t)n_envs, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(P->block_map, bmap.data(), sizeof(int2) * bmap.size(), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(P->prep_map, pmap.data(), sizeof(int4) * pmap.size(), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess)
        ce = cudaMemcpy(P->chunk_first, chunk_first.data(), sizeof(int32_t) * chunk_first.size(), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) { delete P; return fail(CS_ERR_CUDA, "plan upload: %s", cudaGetErrorString(ce)); }
    *plan = P;
    return CS_OK;
}

int cs_plan_create_reduce(int64_t n_envs, const int64_t *capacity, const cs_reduction_params *params, cs_plan **plan) {
    if (!plan) return fail(CS_ERR_VALUE, "null plan pointer");
    *plan = nullptr;
    if (n_envs < 1) return fail(CS_ERR_VALUE, "n_envs must be positive");
    int r = check_params(params);
    if (r) return r;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        r = ensure_tables();
        if (r) return r;
    }
    std::vector<int64_t> cap((size_t)n_envs);
    for (int64_t e = 0; e < n_envs; ++e) {
        if (capacity[e] < 0 || capacity[e] >= ((int64_t)1 << 31)) return fail(CS_ERR_VALUE, "bad capacity");
        cap[(size_t)e] = capacity[e];
    }
    cs_plan *P = new cs_plan();
    P->E = n_envs;
    P->stages = CS_STAGE_REDUCE;
    P->rp.N = params->max_patches; P->rp.K = params->per_patch_cap; P->rp.batch_size = params->batch_size;
    P->rp.has_min_depth = params->has_min_depth; P->rp.cone = params->normal_cone_cos; P->rp.min_depth = params->min_depth;
    r = plan_buffers(P, cap);
    if (r) { delete P; return r; }
    *plan = P;
    return CS_OK;
}

int cs_plan_destroy(cs_plan *plan) {
    delete plan;
    return CS_OK;
}

int cs_plan_device_bytes(cs_plan *plan, int64_t *bytes) {
    if (!plan || !bytes) return fail(CS_ERR_VALUE, "null argument");
    *bytes = plan->device_bytes;
    return CS_OK;
}

int cs_plan_outputs(cs_plan *plan, cs_outputs *out) {
    if (!plan || !out) return fail(CS_ERR_VALUE, "null argument");
    *out = plan->out;
    return CS_OK;
}

static int run_reduce(cs_plan *P, cudaStream_t s) {
    launch_reduce(P->io, P->rp, P->max_batch, s);
    CS_LAUNCHED();
    launch_finalize(P->io, P->rp, g_sms > 0 ? g_sms : 148, s, P->get_fork());
    CS_LAUNCHED();
    return CS_OK;
}

int cs_collide(cs_plan *P, const double *sdf_pose, const double *mesh_pose, int32_t pose_format,
               const double *contact_distance, void *stream) {
    return cs_collide_active(P, sdf_pose, mesh_pose, pose_format, contact_distance, nullptr, stream);
}

int cs_collide_active(cs_plan *P, const double *sdf_pose, const double *mesh_pose, int32_t pose_format,
                      const double *contact_distance, const int32_t *active, void *stream) {
    if (!P || !(P->stages & CS_STAGE_GENERATE)) return fail(CS_ERR_VALUE, "plan has no generate stage");
    if (pose_format != CS_POSE7 && pose_format != CS_POSE12) return fail(CS_ERR_VALUE, "bad pose format");
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t *ev = nullptr;
    if (!P->events.empty()) {
        ev = &P->events[(size_t)(P->timing_step % P->timing_slots) * CS_TIMING_EVENTS];
        ++P->timing_step;
    }
    auto mark = [&](int i) { if (ev) cudaEventRecord(ev[i], s); };
    mark(0);
    launch_env_xf(P->E, P->env_sdf, P->env_mesh, d_sdfs, sdf_pose, mesh_pose, pose_format, contact_distance, P->xf,
                  P->status, P->env_min_depth, P->st.work_count, s, active);
    CS_LAUNCHED();
    mark(1);
    const PlanGrid *ug = P->uniform_sdf ? &P->uniform_grid : nullptr;
    launch_face_prep(P->nblocks, P->prep_map, P->xf, d_sdfs, d_meshes, P->cand_base, P->st, P->max_chunk_verts,
                     P->sample_counter, ug, s, P->uniform_mesh ? &P->uniform_mesh_desc : nullptr);
    CS_LAUNCHED();
    mark(2);
    launch_pgd_wave(g_sms > 0 ? g_sms : 148, P->block_map, P->xf, d_sdfs, d_meshes, P->st,
                    P->sample_counter ? P->sample_counter + 1 : nullptr, ug, s,
                    P->uniform_mesh ? &P->uniform_mesh_desc : nullptr);
    CS_LAUNCHED();
    mark(3);
    launch_compact(P->E, P->xf, P->cand_base, P->block_map, P->chunk_first, P->st, P->cands, P->io.n_cand, s);
    CS_LAUNCHED();
    mark(4);
    if (P->stages & CS_STAGE_REDUCE) {
        launch_reduce(P->io, P->rp, P->max_batch, s);
        CS_LAUNCHED();
        mark(5);
        launch_finalize(P->io, P->rp, g_sms > 0 ? g_sms : 148, s, P->get_fork());
        CS_LAUNCHED();
    } else {
        mark(5);
    }
    mark(6);
    return CS_OK;
}

int cs_plan_timing(cs_plan *P, int32_t slots) {
    if (!P) return fail(CS_ERR_VALUE, "null plan");
    for (cudaEvent_t e : P->events) cudaEventDestroy(e);
    P->events.clear();
    P->timing_step = 0;
    P->timing_slots = slots > 0 ? slots : 0;
    for (int64_t i = 0; i < (int64_t)P->timing_slots * CS_TIMING_EVENTS; ++i) {
        cudaEvent_t e;
        CS_CUDA(cudaEventCreate(&e));
        P->events.push_back(e);
    }
    return CS_OK;
}

int cs_plan_timing_read(cs_plan *P, float *ms, int32_t max_steps, int32_t *n_steps) {
    if (!P || P->events.empty()) return fail(CS_ERR_VALUE, "plan timing is not enabled");
    int64_t n = std::min<int64_t>(P->timing_step, P->timing_slots);
    n = std::min<int64_t>(n, max_steps);
    const int64_t first = P->timing_step - n;
    for (int64_t k = 0; k < n; ++k) {
        cudaEvent_t *ev = &P->events[(size_t)((first + k) % P->timing_slots) * CS_TIMING_EVENTS];
        CS_CUDA(cudaEventSynchronize(ev[CS_TIMING_EVENTS - 1]));
        for (int p = 0; p < CS_TIMING_EVENTS - 1; ++p)
            CS_CUDA(cudaEventElapsedTime(ms + k * CS_TIMING_PHASES + p, ev[p], ev[p + 1]));
        CS_CUDA(cudaEventElapsedTime(ms + k * CS_TIMING_PHASES + CS_TIMING_EVENTS - 1, ev[0], ev[CS_TIMING_EVENTS - 1]));
    }
    *n_steps = (int32_t)n;
    return CS_OK;
}

int cs_plan_count_samples(cs_plan *P, int32_t enable, uint64_t *count) {
    if (!P) return fail(CS_ERR_VALUE, "null plan");
    if (enable) {
        if (!P->counter_buf) {
            int r = P->alloc(&P->counter_buf, CS_SAMPLE_COUNTERS);
            if (r) return r;
        }
        CS_CUDA(cudaMemset(P->counter_buf, 0, sizeof(unsigned long long) * CS_SAMPLE_COUNTERS));
        P->sample_counter = P->counter_buf;
        return CS_OK;
    }
    if (count) {
        if (!P->counter_buf) return fail(CS_ERR_VALUE, "sample counting was never enabled");
        CS_CUDA(cudaDeviceSynchronize());
        CS_CUDA(cudaMemcpy(count, P->counter_buf, sizeof(uint64_t) * CS_SAMPLE_COUNTERS, cudaMemcpyDeviceToHost));
    }
    P->sample_counter = nullptr;
    return CS_OK;
}

int cs_reduce(cs_plan *P, void *stream) {
    if (!P || !(P->stages & CS_STAGE_REDUCE)) return fail(CS_ERR_VALUE, "plan has no reduce stage");
    return run_reduce(P, (cudaStream_t)stream);
}

int cs_collide_host(cs_plan *P, const double *sdf_pose_host, const double *mesh_pose_host, int32_t pose_format,
                    const double *contact_distance_host, float *stats_host, void *stream) {
    if (!P || !(P->stages & CS_STAGE_GENERATE)) return fail(CS_ERR_VALUE, "plan has no generate stage");
    const size_t w = pose_format == CS_POSE12 ? 12 : 7;
    if (!P->in_sdf) {
        int r;
        if ((r = P->alloc(&P->in_sdf, 12 * (size_t)P->E))) return r;
        if ((r = P->alloc(&P->in_mesh, 12 * (size_t)P->E))) return r;
        if ((r = P->alloc(&P->in_cd, (size_t)P->E))) return r;
    }
    cudaStream_t s = (cudaStream_t)stream;
    CS_CUDA(cudaMemcpyAsync(P->in_sdf, sdf_pose_host, sizeof(double) * w * (size_t)P->E, cudaMemcpyHostToDevice, s));
    CS_CUDA(cudaMemcpyAsync(P->in_mesh, mesh_pose_host, sizeof(double) * w * (size_t)P->E, cudaMemcpyHostToDevice, s));
    CS_CUDA(cudaMemcpyAsync(P->in_cd, contact_distance_host, sizeof(double) * (size_t)P->E, cudaMemcpyHostToDevice, s));
    // The step from a CUDA graph (the kernels' launch gaps removed): captured on a plan
    // stream from the second call on, per pose format; eager while phase timing is on or
    // if the capture failed.
    bool replayed = false;
    if (P->events.empty() && !P->host_graph_failed) {
        if ((!P->host_exec || P->host_fmt != pose_format) && P->host_calls >= 1) {
            if (P->host_exec) { cudaGraphExecDestroy(P->host_exec); P->host_exec = nullptr; }
            cudaGraph_t graph = nullptr;
            bool ok = P->host_cap || cudaStreamCreateWithFlags(&P->host_cap, cudaStreamNonBlocking) == cudaSuccess;
            ok = ok && cudaStreamBeginCapture(P->host_cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                const int rc = cs_collide(P, P->in_sdf, P->in_mesh, pose_format, P->in_cd, P->host_cap);
                ok = cudaStreamEndCapture(P->host_cap, &graph) == cudaSuccess && rc == CS_OK && graph;
            }
            ok = ok && cudaGraphInstantiate(&P->host_exec, graph, 0) == cudaSuccess;
            if (graph) cudaGraphDestroy(graph);
            if (!ok) {
                if (P->host_exec) cudaGraphExecDestroy(P->host_exec);
                P->host_exec = nullptr;
                P->host_graph_failed = true;
                cudaGetLastError();  // the failed capture's error is not the caller's
            }
            P->host_fmt = pose_format;
        }
        if (P->host_exec && P->host_fmt == pose_format) {
            CS_CUDA(cudaGraphLaunch(P->host_exec, s));
            replayed = true;
        }
    }
    ++P->host_calls;
    if (!replayed) {
        const int r = cs_collide(P, P->in_sdf, P->in_mesh, pose_format, P->in_cd, stream);
        if (r) return r;
    }
    if (stats_host && (P->stages & CS_STAGE_REDUCE))
        CS_CUDA(cudaMemcpyAsync(stats_host, P->io.stats, sizeof(float) * 4 * (size_t)P->E, cudaMemcpyDeviceToHost, s));
    CS_CUDA(cudaStreamSynchronize(s));
    return CS_OK;
}

// ---------------------------------------------------------------- contact solver

namespace {
int check_sys(int64_t n_sys, int32_t nb, const int64_t *row_off) {
    if (n_sys < 0) return fail(CS_ERR_VALUE, "n_sys must be non-negative");
    if (nb < 1 || nb > SOLVER_MAX_BODIES) return fail(CS_ERR_VALUE, "n_bodies must be in [1, %d]", SOLVER_MAX_BODIES);
    if (n_sys > 0 && !row_off) return fail(CS_ERR_VALUE, "null row_off");
    return CS_OK;
}
}  // namespace

int cs_constraints_build(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, const int64_t *body_a,
                         const int64_t *body_b, const double *point, const double *normal, const double *depth,
                         const double *restitution, const double *slop, const double *ref, const double *w_mat,
                         const double *vel, double h, double bias_factor, double *ra, double *rb, double *tan1,
                         double *tan2, double *kn, double *kt1, double *kt2, double *bias_target,
                         double *restitution_target, void *stream) {
    if (int r = check_sys(n_sys, n_bodies, row_off)) return r;
    const SysRows rows{row_off, 0, nullptr, 0};
    const BuildIO io{body_a, body_b, point, normal, depth, restitution, slop, ref, w_mat, vel, h, bias_factor,
                     ra, rb, tan1, tan2, kn, kt1, kt2, bias_target, restitution_target};
    launch_constraints_build(n_sys, n_bodies, rows, io, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_gauss_seidel_sweeps(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, int64_t iters,
                           const double *w_mat, double *vel, double *imp, const int64_t *body_a,
                           const int64_t *body_b, const double *ra, const double *rb, const double *nrm,
                           const double *tan1, const double *tan2, const double *kn, const double *kt1,
                           const double *kt2, const double *target_vn, const double *mu, double *lam_n,
                           double *lam_t1, double *lam_t2, int32_t with_friction, void *stream) {
    if (int r = check_sys(n_sys, n_bodies, row_off)) return r;
    const SysRows rows{row_off, 0, nullptr, 0};
    const SweepIO io{body_a, body_b, ra, rb, nrm, tan1, tan2, kn, kt1, kt2, mu, lam_t1, lam_t2, w_mat, vel, imp};
    const SweepPhase ph{iters, target_vn, lam_n, with_friction ? 1 : 0};
    launch_sweeps(n_sys, n_bodies, rows, io, &ph, 1, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_body_wrenches(int64_t n_sys, int32_t n_bodies, const int64_t *row_off, const int64_t *body_a,
                     const int64_t *body_b, const double *ra, const double *rb, const double *nrm,
                     const double *tan1, const double *tan2, const double *lam_n, const double *lam_vel,
                     const double *lam_t1, const double *lam_t2, double h, double *out, void *stream) {
    if (int r = check_sys(n_sys, n_bodies, row_off)) return r;
    const SysRows rows{row_off, 0, nullptr, 0};
    const WrenchIO io{body_a, body_b, ra, rb, nrm, tan1, tan2, lam_n, lam_vel, lam_t1, lam_t2, h, out};
    launch_body_wrenches(n_sys, n_bodies, rows, io, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

namespace {
int alloc_rows(cs_plan *P, cs_solver_rows &S, int64_t stride, int64_t R) {
    int r = 0;
    S.stride = stride;
    S.planes = R;
    if ((r = P->alloc(&S.body_a, R)) || (r = P->alloc(&S.body_b, R)) || (r = P->alloc(&S.point, 3 * R)) ||
        (r = P->alloc(&S.normal, 3 * R)) || (r = P->alloc(&S.depth, R)) || (r = P->alloc(&S.mu, R)) ||
        (r = P->alloc(&S.restitution, R)) || (r = P->alloc(&S.slop, R)) || (r = P->alloc(&S.ra, 3 * R)) ||
        (r = P->alloc(&S.rb, 3 * R)) || (r = P->alloc(&S.tan1, 3 * R)) || (r = P->alloc(&S.tan2, 3 * R)) ||
        (r = P->alloc(&S.kn, R)) || (r = P->alloc(&S.kt1, R)) || (r = P->alloc(&S.kt2, R)) ||
        (r = P->alloc(&S.bias_target, R)) || (r = P->alloc(&S.restitution_target, R)) ||
        (r = P->alloc(&S.lam_n, 4 * R)))
        return r;
    S.lam_vel = S.lam_n + R;
    S.lam_t1 = S.lam_n + 2 * R;
    S.lam_t2 = S.lam_n + 3 * R;
    return CS_OK;
}

// rows -> build -> sweeps (position with friction, then velocity) -> wrenches
int solve_rows(cs_plan *P, const cs_solver_rows &S, const SysRows &rows, int64_t n_sys, int nb, bool fixed,
               const double *ref, const double *w_mat, double *vel, double *imp, const cs_solver_params *params,
               double *wrench, cudaStream_t s, double *packed) {
    const BuildIO bio{S.body_a, S.body_b, S.point, S.normal, S.depth, S.restitution, S.slop, ref, w_mat, vel,
                      params->h, params->bias_factor, S.ra, S.rb, S.tan1, S.tan2, S.kn, S.kt1, S.kt2,
                      S.bias_target, S.restitution_target};
    launch_constraints_build(n_sys, nb, rows, bio, s);
    CS_CUDA(cudaMemsetAsync(S.lam_n, 0, sizeof(double) * 4 * (size_t)S.planes, s));
    const SweepIO sio{S.body_a, S.body_b, S.ra, S.rb, S.normal, S.tan1, S.tan2, S.kn, S.kt1, S.kt2, S.mu,
                      S.lam_t1, S.lam_t2, w_mat, vel, imp};
    const SweepPhase ph[2] = {{params->pos_iterations, S.bias_target, S.lam_n, 1},
                              {params->vel_iterations, S.restitution_target, S.lam_vel, 0}};
    if (packed) launch_sweeps_packed(n_sys, nb, rows, sio, ph, 2, packed, s, fixed);
    else launch_sweeps(n_sys, nb, rows, sio, ph, 2, s, fixed);
    const WrenchIO wio{S.body_a, S.body_b, S.ra, S.rb, S.normal, S.tan1, S.tan2, S.lam_n, S.lam_vel, S.lam_t1,
                       S.lam_t2, params->h, wrench};
    launch_body_wrenches(n_sys, nb, rows, wio, s);
    CS_LAUNCHED();
    return CS_OK;
}

int check_solver_params(const cs_solver_params *params) {
    if (!params) return fail(CS_ERR_VALUE, "null argument");
    if (!(params->h > 0.0)) return fail(CS_ERR_VALUE, "h must be positive");
    if (params->pos_iterations < 1) return fail(CS_ERR_VALUE, "pos_iterations must be at least 1");
    if (params->vel_iterations < 0) return fail(CS_ERR_VALUE, "vel_iterations must be non-negative");
    return CS_OK;
}
}  // namespace

int cs_plan_solve(cs_plan *P, const double *ref, const double *w_mat, double *vel, double *imp, const double *mu,
                  const double *restitution, const double *slop, const cs_solver_params *params, double *wrench,
                  void *stream) {
    if (!P || !(P->stages & CS_STAGE_REDUCE)) return fail(CS_ERR_VALUE, "plan has no reduce stage");
    if (!ref || !w_mat || !vel || !imp || !mu || !restitution || !slop || !wrench)
        return fail(CS_ERR_VALUE, "null argument");
    if (int r = check_solver_params(params)) return r;
    const int64_t E = P->E, NK = (int64_t)P->rp.N * P->rp.K, R = (E + 31) / 32 * 32 * NK;
    cs_solver_rows &S = P->srows;
    if (!S.body_a) {
        if (int r = alloc_rows(P, S, NK, R)) return r;
        if (int r = P->alloc(&P->spacked, (size_t)E * NK * 22)) return r;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const SysRows rows{nullptr, NK, P->io.n_kept, R};
    PlanRowsIO pr{P->io.patch_nkept, P->io.n_patch, P->io.kept_point, P->io.kept_normal, P->io.kept_depth, mu,
                  restitution, slop, nullptr, nullptr, nullptr, P->rp.N, P->rp.K, rows, nullptr, S.body_a,
                  S.body_b, S.point, S.normal, S.depth, S.mu, S.restitution, S.slop};
    launch_plan_rows(E, pr, s);
    return solve_rows(P, S, rows, E, 2, true, ref, w_mat, vel, imp, params, wrench, s, P->spacked);
}

int cs_plan_solver_rows(cs_plan *P, cs_solver_rows *rows) {
    if (!P || !rows) return fail(CS_ERR_VALUE, "null argument");
    if (!P->srows.body_a) return fail(CS_ERR_VALUE, "cs_plan_solve has not run on this plan");
    *rows = P->srows;
    return CS_OK;
}

int cs_multipair_solve(cs_plan *P, int64_t n_sys, int32_t nb, const int64_t *slot_off, const int64_t *slot_a,
                       const int64_t *slot_b, int32_t max_slots, const double *ref, const double *w_mat, double *vel,
                       double *imp, const double *mu, const double *restitution, const double *slop,
                       const cs_solver_params *params, double *wrench, void *stream) {
    if (!P || !(P->stages & CS_STAGE_REDUCE)) return fail(CS_ERR_VALUE, "plan has no reduce stage");
    if (n_sys < 1 || max_slots < 1) return fail(CS_ERR_VALUE, "n_sys and max_slots must be positive");
    if (nb < 1 || nb > SOLVER_MAX_BODIES) return fail(CS_ERR_VALUE, "n_bodies must be in [1, %d]", SOLVER_MAX_BODIES);
    if (!slot_off || !slot_a || !slot_b || !ref || !w_mat || !vel || !imp || !mu || !restitution || !slop || !wrench)
        return fail(CS_ERR_VALUE, "null argument");
    if (int r = check_solver_params(params)) return r;
    const int64_t stride = (int64_t)max_slots * P->rp.N * P->rp.K, R = (n_sys + 31) / 32 * 32 * stride;
    cs_solver_rows &S = P->mrows;
    if (S.body_a && (P->mrows_sys != n_sys || S.stride != stride))
        return fail(CS_ERR_VALUE, "a plan serves one multi-pair layout (n_sys / max_slots changed)");
    if (!S.body_a) {
        if (int r = alloc_rows(P, S, stride, R)) return r;
        if (int r = P->alloc(&P->mrow_count, n_sys)) return r;
        if (int r = P->alloc(&P->mpacked, (size_t)n_sys * stride * 22)) return r;
        P->mrows_sys = n_sys;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const SysRows rows{nullptr, stride, P->mrow_count, R};
    PlanRowsIO pr{P->io.patch_nkept, P->io.n_patch, P->io.kept_point, P->io.kept_normal, P->io.kept_depth, mu,
                  restitution, slop, slot_off, slot_a, slot_b, P->rp.N, P->rp.K, rows, P->mrow_count, S.body_a,
                  S.body_b, S.point, S.normal, S.depth, S.mu, S.restitution, S.slop};
    launch_plan_rows(n_sys, pr, s);
    return solve_rows(P, S, rows, n_sys, nb, false, ref, w_mat, vel, imp, params, wrench, s, P->mpacked);
}

int cs_plan_multipair_rows(cs_plan *P, cs_solver_rows *rows, const int32_t **n_rows) {
    if (!P || !rows || !n_rows) return fail(CS_ERR_VALUE, "null argument");
    if (!P->mrows.body_a) return fail(CS_ERR_VALUE, "cs_multipair_solve has not run on this plan");
    *rows = P->mrows;
    *n_rows = P->mrow_count;
    return CS_OK;
}

// ---------------------------------------------------------------- broadphase

int cs_world_aabb(int64_t n, const double *mesh_lo, const double *mesh_hi, const double *pose7, double *lo,
                  double *hi, void *stream) {
    if (n < 0) return fail(CS_ERR_VALUE, "n must be non-negative");
    if (n > 0 && (!mesh_lo || !mesh_hi || !pose7 || !lo || !hi)) return fail(CS_ERR_VALUE, "null argument");
    launch_world_aabb(n, mesh_lo, mesh_hi, pose7, lo, hi, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_broadphase(int64_t n_scenes, const int64_t *body_off, const double *lo, const double *hi, const int64_t *ids,
                  const double *margin, const int64_t *pair_off, int64_t *pairs, int32_t *n_pairs, int32_t *status,
                  void *stream) {
    if (n_scenes < 0) return fail(CS_ERR_VALUE, "n_scenes must be non-negative");
    if (n_scenes > 0 && (!body_off || !lo || !hi || !ids || !margin || !pair_off || !pairs || !n_pairs || !status))
        return fail(CS_ERR_VALUE, "null argument");
    const BroadIO io{body_off, lo, hi, ids, margin, pair_off, pairs, n_pairs, status};
    launch_broadphase(n_scenes, io, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

int cs_pair_slots_active(int64_t n_slots, const int64_t *slot_scene, const int64_t *slot_pair,
                         const int64_t *pair_off, const int64_t *pairs, const int32_t *n_pairs, int32_t *active,
                         void *stream) {
    if (n_slots < 0) return fail(CS_ERR_VALUE, "n_slots must be non-negative");
    launch_pair_slots(n_slots, slot_scene, slot_pair, pair_off, pairs, n_pairs, active, (cudaStream_t)stream);
    CS_LAUNCHED();
    return CS_OK;
}

// ---------------------------------------------------------------- SDF generation

int cs_sdf_generate(const double *vertices, int64_t nv, const int32_t *triangles, int64_t nt, int32_t nx, int32_t ny,
                    int32_t nz, const double origin[3], double voxel, float *values_out) {
    if (!vertices || !triangles || !values_out || !origin) return fail(CS_ERR_VALUE, "null argument");
    if (nx < 2 || ny < 2 || nz < 2) return fail(CS_ERR_VALUE, "grid dims must be at least 2 per axis");
    if (!(voxel > 0.0)) return fail(CS_ERR_VALUE, "voxel must be positive");
    if (nt < 1) return fail(CS_ERR_MESH, "empty mesh");
    for (int64_t i = 0; i < 3 * nt; ++i)
        if (triangles[i] < 0 || triangles[i] >= nv) return fail(CS_ERR_MESH, "triangle index out of range");
    std::string err;
    int code = sdf_generate(vertices, nv, triangles, nt, nx, ny, nz, origin, voxel, values_out, &err);
    if (code) return fail(code, "%s", err.c_str());
    return CS_OK;
}

}  // extern "C"
