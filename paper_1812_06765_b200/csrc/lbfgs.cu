// L-BFGS vector algebra on the device (lbfgs.py:68-181).
//
// The Python driver keeps the reference control flow; every vector operation and
// every reduction it branches on runs here.  Reductions are deterministic: a fixed
// grid of kRedBlocks blocks writes per-block partials, and the last block to finish
// sums them in block order.  Scalars the reference holds as Python floats are kept
// as doubles; vector updates reproduce the reference's dtype rounding
// (python float -> dtype cast, then one dtype multiply and one dtype add).

#include <cooperative_groups.h>

#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"
#include "lbfgs.cuh"

namespace cg = cooperative_groups;

namespace ngf {

constexpr int kRedBlocks = kSMs;  // one block per SM: also co-resident for the cooperative kernel
constexpr int kRedThreads = 256;
constexpr int kNStat = 5;

struct Scratch {
    double* parts = nullptr;         // [2][kRedBlocks][kNStat]
    unsigned int* counter = nullptr;  // last-block counter
};

// One scratch (block partials + last-block counter) per (device, stream): the reductions'
// last-block pattern shares it between launches, so launches on different streams (e.g.
// concurrent registrations) must not share one.
static std::mutex g_scr_mu;
static std::map<std::pair<int, cudaStream_t>, Scratch> g_scr;

static Scratch* scratch(cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_scr_mu);
    Scratch& s = g_scr[{dev, st}];
    if (!s.parts) {
        if (cudaMalloc(&s.parts, 2 * kRedBlocks * kNStat * sizeof(double)) != cudaSuccess) return nullptr;
        if (cudaMalloc(&s.counter, 64) != cudaSuccess) return nullptr;
        cudaMemset(s.counter, 0, 64);
        cudaDeviceSynchronize();
    }
    return &s;
}

template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double (&red)[K][kRedThreads / 32]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) red[k][threadIdx.x >> 5] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < kRedThreads / 32; ++w) s += red[k][w];
            v[k] = s;
        }
    }
}

// Final reduction of the block partials by warp 0 of the last block: NS sums (k < NS)
// and a max (k == NS), lane-strided over the blocks in order, then a butterfly (fixed order).
template <int NS>
__device__ __forceinline__ void final_reduce(const double* parts, int nblocks, double* out) {
    if (threadIdx.x >= 32) return;
    double acc[NS], m = 0.0;
#pragma unroll
    for (int k = 0; k < NS; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 32) {
#pragma unroll
        for (int k = 0; k < NS; ++k) acc[k] += __ldcg(parts + b * kNStat + k);
        m = fmax(m, __ldcg(parts + b * kNStat + NS));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < NS; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NS; ++k) out[k] = acc[k];
        out[NS] = m;
    }
}

// stats: [0] g.d  [1] s.y  [2] s.s  [3] y.y  [4] max|g|
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_stats(const T* __restrict__ g, const T* __restrict__ d,
                                                       const T* __restrict__ s, const T* __restrict__ y,
                                                       int64_t n, double* parts, unsigned int* counter,
                                                       double* out) {
    __shared__ double red[4][kRedThreads / 32];
    __shared__ bool last;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (g) {
            const double gv = (double)g[i];
            if (d) v[0] += gv * (double)d[i];
            mx = fmax(mx, fabs(gv));
        }
        if (s) {
            const double sv = (double)s[i];
            v[2] += sv * sv;
            if (y) v[1] += sv * (double)y[i];
        }
        if (y) {
            const double yv = (double)y[i];
            v[3] += yv * yv;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double redm[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = mx;
    block_sum<4>(v, red);
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) m = fmax(m, redm[w]);
        for (int k = 0; k < 4; ++k) parts[blockIdx.x * kNStat + k] = v[k];
        parts[blockIdx.x * kNStat + 4] = m;
        __threadfence();
        const unsigned int t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        final_reduce<4>(parts, gridDim.x, out);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// x_new = x + dtype(t) * d  (lbfgs.py:122, :137)
template <typename T>
__global__ void k_axpy_step(const T* __restrict__ x, T t, const T* __restrict__ d, T* __restrict__ out,
                            int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __fadd_rn_t(x[i], __fmul_rn_t(t, d[i]));
}

template <typename T>
__global__ void k_sub(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}

// s = x_new - x, y = g_new - g and their stats in one pass (lbfgs.py:145-148, :161-164)
template <typename T>
__device__ __forceinline__ void pair_body(const T* __restrict__ xn, const T* __restrict__ x,
                                          const T* __restrict__ gn, const T* __restrict__ g,
                                          T* __restrict__ s_out, T* __restrict__ y_out, int64_t n,
                                          double* parts, unsigned int* counter, double* out) {
    __shared__ double red[4][kRedThreads / 32];
    __shared__ double redm[kRedThreads / 32];
    __shared__ bool last;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const T sv = xn[i] - x[i];
        const T gv = gn[i];
        const T yv = gv - g[i];
        s_out[i] = sv;
        y_out[i] = yv;
        v[0] += (double)sv * (double)yv;
        v[1] += (double)sv * (double)sv;
        v[2] += (double)yv * (double)yv;
        mx = fmax(mx, fabs((double)gv));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = mx;
    block_sum<4>(v, red);
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) m = fmax(m, redm[w]);
        for (int k = 0; k < 3; ++k) parts[blockIdx.x * kNStat + k] = v[k];
        parts[blockIdx.x * kNStat + 3] = m;
        __threadfence();
        const unsigned int t = atomicAdd(counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        final_reduce<3>(parts, gridDim.x, out);
        if (threadIdx.x == 0) *counter = 0u;
    }
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_pair(const T* __restrict__ xn, const T* __restrict__ x,
                                                      const T* __restrict__ gn, const T* __restrict__ g,
                                                      T* __restrict__ s_out, T* __restrict__ y_out,
                                                      int64_t n, double* parts, unsigned int* counter,
                                                      double* out) {
    pair_body(xn, x, gn, g, s_out, y_out, n, parts, counter, out);
}

// the same with the output pair chosen on the device (graph-driven solver)
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_pair_ind(const T* __restrict__ xn, const T* __restrict__ x,
                                                          const T* __restrict__ gn, const T* __restrict__ g,
                                                          T* const* s_ptr, T* const* y_ptr, int64_t n,
                                                          double* parts, unsigned int* counter, double* out) {
    pair_body(xn, x, gn, g, *s_ptr, *y_ptr, n, parts, counter, out);
}

template <typename T>
__global__ void k_axpy_ind(const T* __restrict__ x, const double* t, const T* __restrict__ d,
                           T* __restrict__ out, int64_t n) {
    const T tt = (T)*t;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __fadd_rn_t(x[i], __fmul_rn_t(tt, d[i]));
}

// grid-wide deterministic sum of one value per thread: block partial -> parts[buf][b],
// grid sync, every block sums the partials in block order (identical result everywhere)
__device__ __forceinline__ double grid_dot(cg::grid_group& grid, double v, double* parts, int buf,
                                           double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        parts[buf * kRedBlocks + blockIdx.x] = s;
    }
    grid.sync();
    // one warp per block sums the block partials: lane-strided in block order, then a
    // butterfly -- the same fixed order in every block, so all blocks agree bit for bit
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) t += __ldcg(parts + buf * kRedBlocks + b);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const double tot = red[0];
    __syncthreads();  // red reused by the next call
    return tot;
}

// one-block variant for short vectors: the same fixed-order sum within the block
__device__ __forceinline__ double block_dot(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    const double tot = red[32];
    __syncthreads();
    return tot;
}

// GRID: cooperative launch over kRedBlocks blocks (long vectors); else one block of
// kSmallThreads threads (no grid synchronisation; vectors up to kSmallN values)
constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallN = 1 << 16;

template <typename T, bool GRID>
__global__ void __launch_bounds__(GRID ? kRedThreads : kSmallThreads) k_two_loop(const TwoLoopArgs<T> a) {
    __shared__ double red[33];
    auto dot = [&](double v, int buf) {
        if constexpr (GRID) {
            cg::grid_group grid = cg::this_grid();
            return grid_dot(grid, v, a.parts, buf, red);
        } else {
            (void)buf;
            return block_dot(v, red);
        }
    };
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    int buf = 0;
    double alpha[kMaxMem];
    // q = g; partial of s_{m-1} . q
    double v = 0.0;
    for (int64_t i = i0; i < a.n; i += st) {
        const T q = a.g[i];
        a.d[i] = q;
        if (a.m > 0) v += (double)a.S[a.m - 1][i] * (double)q;
    }
    // first loop, newest pair first: alpha = rho * (s . q); q -= dtype(alpha) * y
    for (int k = a.m - 1; k >= 0; --k) {
        const double dt = dot(v, buf);
        buf ^= 1;
        alpha[k] = a.rho[k] * dt;
        const T al = (T)alpha[k];
        v = 0.0;
        const bool last = (k == 0);
        const T tg = (T)a.gamma;
        for (int64_t i = i0; i < a.n; i += st) {
            T q = __fsub_rn_t(a.d[i], __fmul_rn_t(al, a.Y[k][i]));
            if (last) {
                q = __fmul_rn_t(q, tg);  // q *= dtype(gamma)
                v += (double)a.Y[0][i] * (double)q;
            } else {
                v += (double)a.S[k - 1][i] * (double)q;
            }
            a.d[i] = q;
        }
    }
    // second loop, oldest pair first: beta = rho * (y . q); q += dtype(alpha - beta) * s
    for (int k = 0; k < a.m; ++k) {
        const double dt = dot(v, buf);
        buf ^= 1;
        const double beta = a.rho[k] * dt;
        const T c = (T)(alpha[k] - beta);
        v = 0.0;
        const bool last = (k == a.m - 1);
        for (int64_t i = i0; i < a.n; i += st) {
            T q = __fadd_rn_t(a.d[i], __fmul_rn_t(c, a.S[k][i]));
            if (last) {
                q = -q;
                v += (double)a.g[i] * (double)q;
            } else {
                v += (double)a.Y[k + 1][i] * (double)q;
            }
            a.d[i] = q;
        }
    }
    if (a.m == 0) {
        // d = -g
        v = 0.0;
        for (int64_t i = i0; i < a.n; i += st) {
            const T q = -a.g[i];
            a.d[i] = q;
            v += (double)a.g[i] * (double)q;
        }
    }
    const double slope = dot(v, buf);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.slope = slope;
}

// Register-resident two-loop (the path used whenever q fits in registers): q stays in
// registers for the whole recursion, and the loads of the next pair's vectors are issued
// before the current reduction, so each of the 2m + 1 sequential steps costs one
// reduction latency instead of a dependent L2 round trip per element.  The reduction
// group is a thread-block cluster (C <= 16 CTAs, partials exchanged through distributed
// shared memory) or, for long vectors, the whole grid of a cooperative launch.  Element
// updates are the same dtype operations as k_two_loop; the dot products are summed in a
// fixed order (warp butterflies, then CTAs in rank order), identical in every CTA.
constexpr int kRvThreads = 512;
constexpr int kRvWarps = kRvThreads / 32;

template <bool GRIDSYNC>
struct RvReducer {
    double* parts;  // grid mode: [2][gridDim.x] block partials
    int C;          // cluster mode: CTAs per cluster
    __device__ __forceinline__ double operator()(double v, int parity, double* wred, double (*cslot)[16],
                                                 double* bcast) const {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) wred[warp] = v;
        __syncthreads();
        double t = 0.0;
        if (warp == 0) {
            t = lane < kRvWarps ? wred[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        }
        if constexpr (GRIDSYNC) {
            if (threadIdx.x == 0) parts[parity * gridDim.x + blockIdx.x] = t;
            cg::this_grid().sync();
            if (warp == 0) {
                double u = 0.0;
                for (int b = lane; b < (int)gridDim.x; b += 32) u += __ldcg(parts + parity * gridDim.x + b);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
                if (lane == 0) *bcast = u;
            }
        } else {
            if (C == 1) {
                if (threadIdx.x == 0) *bcast = t;
            } else {
                cg::cluster_group cl = cg::this_cluster();
                const unsigned me = cl.block_rank();
                if (warp == 0 && lane < C) *cl.map_shared_rank(&cslot[parity][me], lane) = t;
                cl.sync();
                if (warp == 0) {
                    double u = lane < C ? cslot[parity][lane] : 0.0;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
                    if (lane == 0) *bcast = u;
                }
            }
        }
        __syncthreads();
        return *bcast;
    }
};

template <typename T, int VPT, bool GRIDSYNC>
__device__ __forceinline__ void two_loop_rv_body(const TwoLoopArgs<T>& a, int C) {
    __shared__ double wred[32];
    __shared__ double cslot[2][16];
    __shared__ double bcast;
    const RvReducer<GRIDSYNC> red{a.parts, C};
    const int64_t i0 = blockIdx.x * (int64_t)kRvThreads + threadIdx.x;
    const int64_t st = (int64_t)gridDim.x * kRvThreads;
    const int64_t n = a.n;
    T q[VPT], u[VPT], w[VPT];
    auto load = [&](T(&r)[VPT], const T* __restrict__ src) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int64_t i = i0 + j * st;
            r[j] = i < n ? __ldcg(src + i) : T(0);
        }
    };
    int parity = 0;
    double alpha[kMaxMem];
    load(q, a.g);
    double v = 0.0;
    if (a.m > 0) {
        load(w, a.S[a.m - 1]);
#pragma unroll
        for (int j = 0; j < VPT; ++j) v += (double)w[j] * (double)q[j];
    }
    // first loop, newest pair first: alpha = rho * (s . q); q -= dtype(alpha) * y
    for (int k = a.m - 1; k >= 0; --k) {
        load(u, a.Y[k]);
        load(w, k > 0 ? a.S[k - 1] : a.Y[0]);  // in flight during the reduction
        const double dt = red(v, parity, wred, cslot, &bcast);
        parity ^= 1;
        alpha[k] = a.rho[k] * dt;
        const T al = (T)alpha[k];
        const T tg = (T)a.gamma;
        v = 0.0;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            T x = __fsub_rn_t(q[j], __fmul_rn_t(al, u[j]));
            if (k == 0) x = __fmul_rn_t(x, tg);  // q *= dtype(gamma)
            q[j] = x;
            v += (double)w[j] * (double)x;
        }
    }
    // second loop, oldest pair first: beta = rho * (y . q); q += dtype(alpha - beta) * s
    for (int k = 0; k < a.m; ++k) {
        load(u, a.S[k]);
        load(w, k < a.m - 1 ? a.Y[k + 1] : a.g);
        const double dt = red(v, parity, wred, cslot, &bcast);
        parity ^= 1;
        const double beta = a.rho[k] * dt;
        const T c = (T)(alpha[k] - beta);
        const bool last = (k == a.m - 1);
        v = 0.0;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            T x = __fadd_rn_t(q[j], __fmul_rn_t(c, u[j]));
            if (last) x = -x;
            q[j] = x;
            v += (double)w[j] * (double)x;
        }
    }
    if (a.m == 0) {  // d = -g
        v = 0.0;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const T g = q[j];
            q[j] = -g;
            v += (double)g * (double)q[j];
        }
    }
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int64_t i = i0 + j * st;
        if (i < n) a.d[i] = q[j];
    }
    const double slope = red(v, parity, wred, cslot, &bcast);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.slope = slope;
}

template <typename T, int VPT, bool GRIDSYNC>
__global__ void __launch_bounds__(kRvThreads) k_two_loop_rv(const TwoLoopArgs<T> a, int C) {
    two_loop_rv_body<T, VPT, GRIDSYNC>(a, C);
}

// arguments in device memory, rewritten by the graph-driven solver between launches
template <typename T, int VPT>
__global__ void __launch_bounds__(kRvThreads) k_two_loop_rv_ind(const TwoLoopArgs<T>* __restrict__ ap, int C) {
    two_loop_rv_body<T, VPT, false>(*ap, C);
}

template <typename T, int VPT>
int launch_rv(const TwoLoopArgs<T>& a, int C, bool grid, cudaStream_t s) {
    if (grid) {
        TwoLoopArgs<T> aa = a;
        int cc = 1;
        void* args[] = {&aa, &cc};
        g_launches.fetch_add(1, std::memory_order_relaxed);
        NGF_CUDA(cudaLaunchCooperativeKernel((const void*)k_two_loop_rv<T, VPT, true>, dim3(kRedBlocks),
                                             dim3(kRvThreads), args, 0, s));
        return 0;
    }
    // once per instantiation (thread-safe static initialisation)
    static const cudaError_t attr =
        cudaFuncSetAttribute(k_two_loop_rv<T, VPT, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    NGF_CUDA(attr);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kRvThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    NGF_CUDA(cudaLaunchKernelEx(&cfg, k_two_loop_rv<T, VPT, false>, a, C));
    return 0;
}

// Register-resident path if q fits (<= 16 values per thread: more spills); -1 if not.
template <typename T>
int two_loop_rv(const TwoLoopArgs<T>& a, cudaStream_t s) {
    const int64_t n = a.n;
    constexpr int kVmax = 16;
    const char* env = std::getenv("NGF_TWO_LOOP");
    if (env && std::atoi(env) == 0) return -1;
    // smallest cluster giving <= 8 values per thread, else 16 CTAs, else the whole grid
    int C = 1;
    while (C < 16 && (int64_t)C * kRvThreads * 8 < n) C *= 2;
    bool grid = false;
    int64_t threads = (int64_t)C * kRvThreads;
    if ((n + threads - 1) / threads > kVmax) {
        grid = true;
        threads = (int64_t)kRedBlocks * kRvThreads;
        if ((n + threads - 1) / threads > kVmax) return -1;
    }
    const int64_t need = (n + threads - 1) / threads;
    int vpt = 1;
    while (vpt < need) vpt *= 2;
    switch (vpt) {
        case 1: return launch_rv<T, 1>(a, C, grid, s);
        case 2: return launch_rv<T, 2>(a, C, grid, s);
        case 4: return launch_rv<T, 4>(a, C, grid, s);
        case 8: return launch_rv<T, 8>(a, C, grid, s);
        case 16: return launch_rv<T, 16>(a, C, grid, s);
        default: return -1;
    }
}

template <typename T>
int two_loop_impl(const void* const* S, const void* const* Y, const double* rho, double gamma, int m,
                  const void* g, void* d, int64_t n, double* slope, cudaStream_t s) {
    if (m < 0 || m > kMaxMem) return NGF_EARG;
    Scratch* sc = scratch(s);
    if (!sc) return NGF_ENOMEM;
    TwoLoopArgs<T> a;
    for (int k = 0; k < m; ++k) {
        a.S[k] = (const T*)S[k];
        a.Y[k] = (const T*)Y[k];
        a.rho[k] = rho[k];
    }
    a.gamma = gamma;
    a.m = m;
    a.g = (const T*)g;
    a.d = (T*)d;
    a.n = n;
    a.parts = sc->parts;
    a.slope = slope;
    const int rv = two_loop_rv<T>(a, s);
    if (rv >= 0) return rv;
    if (n <= kSmallN) {
        NGF_LAUNCH((k_two_loop<T, false>), 1, kSmallThreads, 0, s, a);
        NGF_CHECK_LAUNCH();
        return 0;
    }
    void* args[] = {&a};
    g_launches.fetch_add(1, std::memory_order_relaxed);
    NGF_CUDA(cudaLaunchCooperativeKernel((const void*)k_two_loop<T, true>, dim3(kRedBlocks), dim3(kRedThreads),
                                         args, 0, s));
    return 0;
}

// ---- device-argument launchers for the graph-driven solver (solver_graph.cu)

static void rv_shape(int64_t n, int& C, int& vpt) {
    C = 1;
    while (C < 16 && (int64_t)C * kRvThreads * 8 < n) C *= 2;
    const int64_t threads = (int64_t)C * kRvThreads;
    const int64_t need = (n + threads - 1) / threads;
    vpt = 1;
    while (vpt < need) vpt *= 2;
}

template <typename T, int VPT>
static int launch_rv_ind(const TwoLoopArgs<T>* ap, int C, cudaStream_t s) {
    static const cudaError_t attr =
        cudaFuncSetAttribute(k_two_loop_rv_ind<T, VPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    NGF_CUDA(attr);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kRvThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    NGF_CUDA(cudaLaunchKernelEx(&cfg, k_two_loop_rv_ind<T, VPT>, ap, C));
    return 0;
}

template <typename T>
int two_loop_dev_launch(const TwoLoopArgs<T>* ap, int64_t n, cudaStream_t s) {
    if (n > kTwoLoopClusterMaxN) return NGF_EARG;
    int C, vpt;
    rv_shape(n, C, vpt);
    switch (vpt) {
        case 1: return launch_rv_ind<T, 1>(ap, C, s);
        case 2: return launch_rv_ind<T, 2>(ap, C, s);
        case 4: return launch_rv_ind<T, 4>(ap, C, s);
        case 8: return launch_rv_ind<T, 8>(ap, C, s);
        case 16: return launch_rv_ind<T, 16>(ap, C, s);
        default: return NGF_EARG;
    }
}

template <typename T>
int pair_dev_launch(const T* xn, const T* x, const T* gn, const T* g, T* const* s_ptr, T* const* y_ptr,
                    int64_t n, double* out, cudaStream_t s, cudaStream_t owner) {
    Scratch* sc = scratch(owner);
    if (!sc) return NGF_ENOMEM;
    NGF_LAUNCH(k_pair_ind<T>, kRedBlocks, kRedThreads, 0, s, xn, x, gn, g, s_ptr, y_ptr, n, sc->parts,
               sc->counter, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int axpy_dev_launch(const T* x, const double* t, const T* d, T* out, int64_t n, cudaStream_t s) {
    NGF_LAUNCH(k_axpy_ind<T>, blocks_for(n, 256), 256, 0, s, x, t, d, out, n);
    NGF_CHECK_LAUNCH();
    return 0;
}

double* lbfgs_parts(cudaStream_t owner) {
    Scratch* sc = scratch(owner);
    return sc ? sc->parts : nullptr;
}

template int two_loop_dev_launch<float>(const TwoLoopArgs<float>*, int64_t, cudaStream_t);
template int two_loop_dev_launch<double>(const TwoLoopArgs<double>*, int64_t, cudaStream_t);
template int pair_dev_launch<float>(const float*, const float*, const float*, const float*, float* const*,
                                    float* const*, int64_t, double*, cudaStream_t, cudaStream_t);
template int pair_dev_launch<double>(const double*, const double*, const double*, const double*,
                                     double* const*, double* const*, int64_t, double*, cudaStream_t,
                                     cudaStream_t);
template int axpy_dev_launch<float>(const float*, const double*, const float*, float*, int64_t, cudaStream_t);
template int axpy_dev_launch<double>(const double*, const double*, const double*, double*, int64_t,
                                     cudaStream_t);

}  // namespace ngf

using namespace ngf;

extern "C" {

int ngf_vec_dot(int dtype, const void* a, const void* b, int64_t n, double* out_dev, void* stream) {
    // out_dev[0..4] receives the stats layout; [0] = a . b
    return ngf_vec_stats(dtype, a, b, nullptr, nullptr, n, out_dev, stream);
}

int ngf_vec_stats(int dtype, const void* g, const void* d, const void* s, const void* y, int64_t n,
                  double* out_dev, void* stream) {
    if (!out_dev || n < 0) return NGF_EARG;
    cudaStream_t st = as_stream(stream);
    Scratch* sc = scratch(st);
    if (!sc) return NGF_ENOMEM;
    if (dtype == NGF_F32)
        NGF_LAUNCH(k_stats<float>, kRedBlocks, kRedThreads, 0, st, (const float*)g, (const float*)d,
                   (const float*)s, (const float*)y, n, sc->parts, sc->counter, out_dev);
    else if (dtype == NGF_F64)
        NGF_LAUNCH(k_stats<double>, kRedBlocks, kRedThreads, 0, st, (const double*)g, (const double*)d,
                   (const double*)s, (const double*)y, n, sc->parts, sc->counter, out_dev);
    else
        return NGF_EARG;
    NGF_CHECK_LAUNCH();
    return 0;
}

int ngf_vec_axpy_step(int dtype, const void* x, double t, const void* d, void* out, int64_t n,
                      void* stream) {
    if (!x || !d || !out || n < 0) return NGF_EARG;
    cudaStream_t st = as_stream(stream);
    if (dtype == NGF_F32)
        NGF_LAUNCH(k_axpy_step<float>, blocks_for(n, 256), 256, 0, st, (const float*)x, (float)t,
                   (const float*)d, (float*)out, n);
    else if (dtype == NGF_F64)
        NGF_LAUNCH(k_axpy_step<double>, blocks_for(n, 256), 256, 0, st, (const double*)x, t,
                   (const double*)d, (double*)out, n);
    else
        return NGF_EARG;
    NGF_CHECK_LAUNCH();
    return 0;
}

int ngf_vec_sub(int dtype, const void* a, const void* b, void* out, int64_t n, void* stream) {
    if (!a || !b || !out || n < 0) return NGF_EARG;
    cudaStream_t st = as_stream(stream);
    if (dtype == NGF_F32)
        NGF_LAUNCH(k_sub<float>, blocks_for(n, 256), 256, 0, st, (const float*)a, (const float*)b,
                   (float*)out, n);
    else if (dtype == NGF_F64)
        NGF_LAUNCH(k_sub<double>, blocks_for(n, 256), 256, 0, st, (const double*)a, (const double*)b,
                   (double*)out, n);
    else
        return NGF_EARG;
    NGF_CHECK_LAUNCH();
    return 0;
}

int ngf_lbfgs_pair(int dtype, const void* x_new, const void* x, const void* g_new, const void* g,
                   void* s_out, void* y_out, int64_t n, double* out_dev, void* stream) {
    if (!x_new || !x || !g_new || !g || !s_out || !y_out || !out_dev || n < 0) return NGF_EARG;
    cudaStream_t st = as_stream(stream);
    Scratch* sc = scratch(st);
    if (!sc) return NGF_ENOMEM;
    if (dtype == NGF_F32)
        NGF_LAUNCH(k_pair<float>, kRedBlocks, kRedThreads, 0, st, (const float*)x_new, (const float*)x,
                   (const float*)g_new, (const float*)g, (float*)s_out, (float*)y_out, n, sc->parts,
                   sc->counter, out_dev);
    else if (dtype == NGF_F64)
        NGF_LAUNCH(k_pair<double>, kRedBlocks, kRedThreads, 0, st, (const double*)x_new,
                   (const double*)x, (const double*)g_new, (const double*)g, (double*)s_out,
                   (double*)y_out, n, sc->parts, sc->counter, out_dev);
    else
        return NGF_EARG;
    NGF_CHECK_LAUNCH();
    return 0;
}

int ngf_lbfgs_two_loop(int dtype, const void* const* S, const void* const* Y, const double* host_rho,
                       double gamma, int m, const void* g, void* d, int64_t n, double* slope_dev,
                       void* stream) {
    if (!g || !d || !slope_dev || n < 0 || m < 0 || (m > 0 && (!S || !Y || !host_rho)))
        return NGF_EARG;
    cudaStream_t st = as_stream(stream);
    if (dtype == NGF_F32) return two_loop_impl<float>(S, Y, host_rho, gamma, m, g, d, n, slope_dev, st);
    if (dtype == NGF_F64) return two_loop_impl<double>(S, Y, host_rho, gamma, m, g, d, n, slope_dev, st);
    return NGF_EARG;
}

}  // extern "C"
