// Shared definitions for libngfb200 (sm_100a).  See include/ngf_b200.h for the ABI.
#pragma once
#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/ngf_b200.h"

namespace ngf {

extern std::atomic<int64_t> g_launches;

// Stream-ordered pool allocations for plans and levels (plan.cu); 0 or NGF_ENOMEM.
int dev_alloc(void** ptr, size_t bytes);
void dev_free(void* ptr);

// Host-buffer transfers (hostio.cu): staged through page-locked memory by the copy
// threads unless the host side is already page-locked.  host_upload is asynchronous
// (the source may be reused on return); host_download returns once dst holds the data.
bool host_is_pinned(const void* p);
int host_upload(void* dst_dev, const void* src, size_t bytes, cudaStream_t s);
int host_download(void* dst, const void* src_dev, size_t bytes, cudaStream_t s);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Count every kernel launch issued by the library (bench.py reports them).
#define NGF_LAUNCH(kernel, grid, block, smem, stream, ...)                         \
    do {                                                                            \
        ::ngf::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                 \
    } while (0)

// Launch with programmatic dependent launch (the kernel may start while the previous
// kernel in the stream drains; it must execute griddepcontrol.wait before touching what
// that kernel writes or reads).  Plain launch while the stream is being captured.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    ::ngf::g_launches.fetch_add(1, std::memory_order_relaxed);
    static const bool pdl_off = std::getenv("NGF_NO_PDL") != nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (pdl_off || cap != cudaStreamCaptureStatusNone) {
        k<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

#define NGF_CHECK_LAUNCH()                                                          \
    do {                                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess) return (int)e_;                                      \
    } while (0)

#define NGF_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) return (int)e_;                                      \
    } while (0)

// Number of SMs on a B200; grids of grid-stride kernels are multiples of this.
constexpr int kSMs = 148;

// Kernel-side view of a grid in the working dtype T.
template <typename T>
struct GridK {
    int nx, ny, nz;
    T hx, hy, hz;       // spacing cast to the working dtype (numpy dtype.type(h))
    T ox, oy, oz;       // origin cast to the working dtype (NEP 50 weak python float)
    double dhx, dhy, dhz, dox, doy, doz;  // exact f64 metadata
    __host__ __device__ int64_t n() const { return (int64_t)nx * ny * nz; }
};

template <typename T>
inline GridK<T> make_gridk(const ngf_grid_t& g) {
    GridK<T> k;
    k.nx = (int)g.dims[0];
    k.ny = (int)g.dims[1];
    k.nz = (int)g.dims[2];
    k.hx = (T)g.spacing[0];
    k.hy = (T)g.spacing[1];
    k.hz = (T)g.spacing[2];
    k.ox = (T)g.origin[0];
    k.oy = (T)g.origin[1];
    k.oz = (T)g.origin[2];
    k.dhx = g.spacing[0];
    k.dhy = g.spacing[1];
    k.dhz = g.spacing[2];
    k.dox = g.origin[0];
    k.doy = g.origin[1];
    k.doz = g.origin[2];
    return k;
}

inline bool grid_ok(const ngf_grid_t* g) {
    if (!g) return false;
    for (int a = 0; a < 3; ++a) {
        if (g->dims[a] < 1 || g->dims[a] > (1 << 20)) return false;
        if (!(g->spacing[a] > 0)) return false;
    }
    return true;
}

inline int64_t grid_n(const ngf_grid_t& g) { return g.dims[0] * g.dims[1] * g.dims[2]; }

inline unsigned blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > (int64_t)kSMs * 64) b = (int64_t)kSMs * 64;  // grid-stride beyond this
    return (unsigned)b;
}

// Device-side plan for one axis: image index -> (i0, w1) and gather rows.
struct AxisDev {
    int ni, nd, width;
    const int32_t* i0;     // [ni]
    const float* w1f;      // [ni]  f32(w1)
    const double* w1d;     // [ni]
    const int32_t* start;  // [nd]
    const float* wf;       // [nd*width] f32(weights)
    const double* wd;      // [nd*width]
};

template <typename T> __device__ __forceinline__ const T* w1_of(const AxisDev& a);
template <> __device__ __forceinline__ const float* w1_of<float>(const AxisDev& a) { return a.w1f; }
template <> __device__ __forceinline__ const double* w1_of<double>(const AxisDev& a) { return a.w1d; }
template <typename T> __device__ __forceinline__ const T* wts_of(const AxisDev& a);
template <> __device__ __forceinline__ const float* wts_of<float>(const AxisDev& a) { return a.wf; }
template <> __device__ __forceinline__ const double* wts_of<double>(const AxisDev& a) { return a.wd; }

// correctly rounded single operations (no contraction), dtype-generic
__device__ __forceinline__ float __fadd_rn_t(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double __fadd_rn_t(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float __fsub_rn_t(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double __fsub_rn_t(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float __fmul_rn_t(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double __fmul_rn_t(double a, double b) { return __dmul_rn(a, b); }

template <typename T> inline const T* w1_host_sel(const AxisDev& a);
template <> inline const float* w1_host_sel<float>(const AxisDev& a) { return a.w1f; }
template <> inline const double* w1_host_sel<double>(const AxisDev& a) { return a.w1d; }

}  // namespace ngf

struct ngf_plan;
namespace ngf {
int plan_upload(ngf_plan* p);
// Copy host -> device and wait until the bytes have LANDED.  A plain cudaMemcpy from
// pageable memory returns once the data is staged, with the DMA still queued on the
// legacy stream, which the (non-blocking) work streams do not wait for: a kernel on
// another stream could read the destination before it is written.
int upload_blocking(void* dst, const void* src, size_t bytes);  // lazily create the plan's device arrays (plan.cu)
}

// Opaque handle layouts (host side).
struct ngf_plan {
    ngf_grid_t def_grid, img_grid;
    int width[3];
    int n_img[3], n_def[3];
    // host copies
    int32_t* h_i0[3];
    double* h_w1[3];
    int32_t* h_start[3];
    int32_t* h_counts[3];
    double* h_w[3];
    // device blob holding all device arrays
    void* d_blob;
    ngf::AxisDev axes[3];
    // workspace for P^T (x/y stage result, 3 * nz_img * ny_def * nx_def doubles)
    void* d_tmp;
    size_t tmp_bytes;
    // completion of the plan's last launch (ngf_prolong), so destroying it waits for that
    // work only, not the whole device (concurrent registrations); `idle` is set by an
    // owner that has already waited (the level)
    cudaEvent_t done;
    int idle;
};

namespace ngf {
// record `ev` on `s` unless `s` is being captured (event records are not allowed in
// conditional graph bodies, and a captured launch completes with the graph)
inline void record_done(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone)
        cudaEventRecord(ev, s);
}
}  // namespace ngf
