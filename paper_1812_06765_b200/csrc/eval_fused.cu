// Fused NGF objective/gradient evaluation for sm_100a: host dispatch of the march
// (fused_march.cuh, compiled per variant in march_v<n>.cu) and the post-march kernel.

#include <cstdlib>
#include <type_traits>
#include <vector>

#include "fused_cfg.cuh"
#include "march_lean.cuh"

namespace ngf {

// ------------------------------------------------------------------ reduce + curvature

// One kernel after the march: grad = grad D (fixed-order sum of the covering tiles'
// partials) + alpha * vol * L^T L u (curvature.py:74-81), the per-block partial sums of
// (L u)^2, and -- in the last block to finish -- the fixed-order totals J, D, S.
// Grid: x/y tiles of 32 x 8 deformation nodes, blockIdx.z = comp * (chunks of the launch)
// + z chunk - pc0; a launch may cover a range of the chunks (pipelined host evaluation), the
// block index and the finished-block count are over all of them.
template <typename T>
struct PostArgs {
    GridK<T> g;
    FusedPlan fp;
    const T* partial;  // null: no grad D term (curvature added to an all-reduced grad D)
    const T* y;        // null: no curvature term (z-slab partial)
    T vol, alpha;
    T* grad;
    int accumulate;    // grad += ... instead of grad = ...
    const double* dpart;
    int nd;
    double* spart;
    int* flag;         // [0] non-finite y seen, [1] finished-block counter
    double half_hbar, half_vol, dalpha;
    double* out;
    int mode;          // 0 full, 1 slab partial, 2 add curvature (see post_finalize)
    int nchunk;        // z chunks of kPostKZ planes per component
    int pc0;           // first z chunk of this launch (grid z = 3 x its chunk count)
    int count;         // blocks counted for the totals: all post blocks of the evaluation
    T ihx2, ihy2, ihz2;  // 1 / h^2 in the working dtype (curvature.py:28-29)
};

template <typename T>
__device__ __forceinline__ T ident(double o, double h, int i) {
    return (T)(o + h * (double)i);  // identity_field_array: f64 centres cast (geometry.py:148-155)
}

// fixed-order totals, reduced by one block (256 threads, strided then warp tree):
// mode 0: J = D + alpha S from both partial sets; 1: D only (slab partial, J = D, S = 0);
// 2: D already in out[1] (all-reduced over slabs), S from spart
template <typename T>
__device__ void post_finalize(const PostArgs<T>& p, int ns) {
    __shared__ double red[2][32];
    const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
    double a = 0.0, b = 0.0;
#pragma unroll 8
    for (int t = tid; t < p.nd; t += nt) a += __ldcg(p.dpart + t);
    if (p.mode != 1) {
#pragma unroll 8
        for (int t = tid; t < ns; t += nt) b += __ldcg(p.spart + t);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = a;
        red[1][tid >> 5] = b;
    }
    __syncthreads();
    if (tid == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < (nt >> 5); ++w) {
            sa += red[0][w];
            sb += red[1][w];
        }
        const double D = p.mode == 2 ? p.out[1] : (double)((T)p.half_hbar * (T)sa);
        const double S = p.mode == 1 ? 0.0 : (double)((T)p.half_vol * (T)sb);
        // a non-finite trial point gives J = inf (objective.py:55-57)
        if (p.mode == 1) {
            p.out[0] = D;
        } else {
            const int bad = atomicOr(p.flag, 0);
            p.out[0] = bad ? INFINITY : D + p.dalpha * S;
            p.flag[0] = 0;
        }
        p.out[1] = D;
        p.out[2] = S;
        p.flag[1] = 0;  // re-arm the block counter for the next launch
    }
}

template <typename T>
__device__ __forceinline__ T d2t_at(T lm, T l0, T lp, int i, int n, T ih2) {
    // (L^T w)_i of the 1-D second difference with zero face rows (curvature.py:33-43)
    if (n < 3) return (T)0;
    T o = (T)0;
    if (i <= n - 3) o += lp;
    if (i >= 1 && i <= n - 2) o -= (T)2 * l0;
    if (i >= 2) o += lm;
    return o * ih2;
}

// k_post: one block = a 32 x 8 tile of deformation nodes on KZ consecutive planes of one
// component.  All global loads -- the slot masks, the covering slots' partials and
// u = y - id on the 36 x 12 x (KZ + 4) neighbourhood -- are issued before the first
// barrier, so a block costs about two memory round trips; L u is then formed once per
// node of the 34 x 10 x (KZ + 2) tile in shared memory.
// k_post: one block = a 32 x 8 tile of deformation nodes on KZ consecutive planes of one
// component.  u = y - id on the 36 x 12 x (KZ + 4) neighbourhood and the cover lists are
// loaded and L u is formed (once per node of the 34 x 10 x (KZ + 2) tile) before the
// kernel waits for the fused march (programmatic dependent launch, so this part overlaps
// the march's last wave); then the covering tiles' partials of all KZ planes are loaded
// together and summed in a fixed order.
constexpr int kPostUX = 36, kPostUY = 12, kPostLX = 34, kPostLY = 10;

template <typename T>
__device__ __forceinline__ T cover_sum_loop(const FusedPlan& fp, const T* __restrict__ partial, int comp,
                                            int i, int j, int k) {
    // general cover lists (short fused z chunks, tiny tiles): fixed order az, ay, ax
    const int win = fp.wz * fp.wy * fp.wx;
    const int32_t* gx = fp.cov_x + i * kCover * 2;
    const int32_t* gy = fp.cov_y + j * kCover * 2;
    const int32_t* gz = fp.cov_z + k * kCover * 2;
    T gd = (T)0;
    for (int az = 0; az < kCover && gz[2 * az] >= 0; ++az)
        for (int ay = 0; ay < kCover && gy[2 * ay] >= 0; ++ay) {
            const int rowc = (gz[2 * az] * fp.nty + gy[2 * ay]) * fp.ntx;
            const int rowo = (gz[2 * az + 1] * fp.wy + gy[2 * ay + 1]) * fp.wx;
            for (int ax = 0; ax < kCover && gx[2 * ax] >= 0; ++ax)
                gd += __ldcg(partial + ((size_t)(rowc + gx[2 * ax]) * 3 + comp) * win + rowo + gx[2 * ax + 1]);
        }
    return gd;
}

template <typename T>
__global__ void __launch_bounds__(256, 3) k_post(const __grid_constant__ PostArgs<T> p) {
    constexpr int KZ = kPostKZ, NU = KZ + 4, NL = KZ + 2;
    constexpr int UPT = (kPostUX * kPostUY + 255) / 256;  // u items per thread and plane
    constexpr int LPT = (kPostLX * kPostLY + 255) / 256;  // L items per thread and plane
    __shared__ T us[NU][kPostUY][kPostUX];
    __shared__ T ls[NL][kPostLY][kPostLX];
    __shared__ long long zsh[KZ][4];  // first four z covers of each plane: partial offset or -1
    __shared__ int zslow[KZ];         // plane with more than four z covers
    __shared__ double red[8];
    __shared__ int last;
    const GridK<T>& g = p.g;
    const FusedPlan& fp = p.fp;
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int nblk = gridDim.x * gridDim.y * 3 * p.nchunk;  // (L u)^2 partials of all launches
    const int pcn = gridDim.z / 3;
    const int comp = blockIdx.z / pcn, chunk = p.pc0 + (blockIdx.z - comp * pcn);
    const int bid = ((comp * p.nchunk + chunk) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 8;
    const int k0 = chunk * KZ;
    const int i = x0 + threadIdx.x, j = y0 + threadIdx.y;
    const bool mine = i < g.nx && j < g.ny;
    const unsigned m = (unsigned)g.nx * g.ny * g.nz;
    const T* yc = p.y ? p.y + (size_t)comp * m : nullptr;
    const int win = fp.wz * fp.wy * fp.wx;

    // ---- (1) cover lists: z covers are block-uniform (smem), x / y covers per thread
    if (p.partial && tid < KZ) {
        const int k = k0 + tid;
        long long o[4] = {-1, -1, -1, -1};
        int slow = 0;
        if (k < g.nz) {
            const int32_t* c = fp.cov_z + k * kCover * 2;
            const int4 v0 = __ldg(reinterpret_cast<const int4*>(c)), v1 = __ldg(reinterpret_cast<const int4*>(c) + 1);
            const int zt[4] = {v0.x, v0.z, v1.x, v1.z}, zo[4] = {v0.y, v0.w, v1.y, v1.w};
            const long long plane = (long long)fp.nty * fp.ntx * 3 * win;
#pragma unroll
            for (int a = 0; a < 4; ++a)
                if (zt[a] >= 0) o[a] = zt[a] * plane + (long long)zo[a] * fp.wy * fp.wx;
            slow = __ldg(c + 8) >= 0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) zsh[tid][a] = o[a];
        zslow[tid] = slow;
    }
    int bxy[2][2];  // ((y tile * ntx + x tile) * 3 + comp) * win + window offset, or -1
    bool xyslow = false;
    if (p.partial && mine) {
        const int4 xv = __ldg(reinterpret_cast<const int4*>(fp.cov_x + i * kCover * 2));
        const int4 yv = __ldg(reinterpret_cast<const int4*>(fp.cov_y + j * kCover * 2));
        xyslow = __ldg(fp.cov_x + i * kCover * 2 + 4) >= 0 || __ldg(fp.cov_y + j * kCover * 2 + 4) >= 0;
        const int cxt[2] = {xv.x, xv.z}, cxo[2] = {xv.y, xv.w};
        const int cyt[2] = {yv.x, yv.z}, cyo[2] = {yv.y, yv.w};
#pragma unroll
        for (int ay = 0; ay < 2; ++ay)
#pragma unroll
            for (int ax = 0; ax < 2; ++ax)
                bxy[ay][ax] = (cyt[ay] >= 0 && cxt[ax] >= 0)
                                  ? ((cyt[ay] * fp.ntx + cxt[ax]) * 3 + comp) * win + cyo[ay] * fp.wx + cxo[ax]
                                  : -1;
    }

    // ---- (2) u = y - id on planes k0-2 .. k0+KZ+1 (clamped; out-of-grid values unused)
    double acc = 0.0;
    bool bad = false;
    if (yc) {
        const double o = comp == 0 ? g.dox : (comp == 1 ? g.doy : g.doz);
        const double h = comp == 0 ? g.dhx : (comp == 1 ? g.dhy : g.dhz);
        int uoff[UPT];
        T idr[UPT];
#pragma unroll
        for (int r = 0; r < UPT; ++r) {
            const int t = min(tid + r * 256, kPostUX * kPostUY - 1);
            const int ey = t / kPostUX, ex = t - ey * kPostUX;
            const int a = min(max(x0 - 2 + ex, 0), g.nx - 1), b = min(max(y0 - 2 + ey, 0), g.ny - 1);
            uoff[r] = b * g.nx + a;
            idr[r] = ident<T>(o, h, comp == 0 ? a : b);
        }
        T uv[NU][UPT];
#pragma unroll
        for (int q = 0; q < NU; ++q) {
            const int zc = min(max(k0 - 2 + q, 0), g.nz - 1);
            const T* yp = yc + (unsigned)zc * (unsigned)(g.nx * g.ny);
#pragma unroll
            for (int r = 0; r < UPT; ++r) uv[q][r] = __ldg(yp + uoff[r]);
        }
#pragma unroll
        for (int q = 0; q < NU; ++q) {
            const T idz = ident<T>(o, h, min(max(k0 - 2 + q, 0), g.nz - 1));
#pragma unroll
            for (int r = 0; r < UPT; ++r) {
                const int t = tid + r * 256;
                if (t < kPostUX * kPostUY) (&us[q][0][0])[t] = uv[q][r] - (comp == 2 ? idz : idr[r]);
            }
        }
    }
    __syncthreads();

    // ---- (3) L u on planes k0-1 .. k0+KZ over the 34 x 10 tile: second differences x, y, z
    // with zero rows at the faces (curvature.py:20-30)
    if (yc) {
#pragma unroll
        for (int r = 0; r < LPT; ++r) {
            const int t = tid + r * 256;
            if (t < kPostLX * kPostLY) {
                const int ly = t / kPostLX, lx = t - ly * kPostLX;
                const int a = x0 - 1 + lx, b = y0 - 1 + ly;
                const bool fx = g.nx >= 3 && a > 0 && a < g.nx - 1, fy = g.ny >= 3 && b > 0 && b < g.ny - 1;
                const int ux = lx + 1, uy = ly + 1;
#pragma unroll
                for (int q = 0; q < NL; ++q) {
                    const int z = k0 - 1 + q, uz = q + 1;
                    const T c = us[uz][uy][ux];
                    T lap = (T)0;
                    if (fx) lap += (us[uz][uy][ux + 1] - (T)2 * c + us[uz][uy][ux - 1]) * p.ihx2;
                    if (fy) lap += (us[uz][uy + 1][ux] - (T)2 * c + us[uz][uy - 1][ux]) * p.ihy2;
                    if (g.nz >= 3 && z > 0 && z < g.nz - 1)
                        lap += (us[uz + 1][uy][ux] - (T)2 * c + us[uz - 1][uy][ux]) * p.ihz2;
                    ls[q][ly][lx] = lap;
                }
            }
        }
        __syncthreads();
    }

    // ---- (4) the fused march's outputs are needed from here on (programmatic dependent
    // launch: everything above overlaps the march's tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the covering tiles' partials of the KZ planes: first two covers per axis, all loads
    // in flight together (fixed order az, ay, ax)
    T pv[KZ][2][2][2];
    if (p.partial && mine && !xyslow) {
#pragma unroll
        for (int q = 0; q < KZ; ++q)
#pragma unroll
            for (int az = 0; az < 2; ++az) {
                const long long zo = zsh[q][az];
#pragma unroll
                for (int ay = 0; ay < 2; ++ay)
#pragma unroll
                    for (int ax = 0; ax < 2; ++ax)
                        pv[q][az][ay][ax] = (zo >= 0 && bxy[ay][ax] >= 0) ? __ldcg(p.partial + zo + bxy[ay][ax]) : (T)0;
            }
    }

    // ---- (5) outputs
    T gdp[KZ];
#pragma unroll
    for (int q = 0; q < KZ; ++q) gdp[q] = (T)0;
    if (p.partial && mine) {
        if (xyslow) {
#pragma unroll
            for (int q = 0; q < KZ; ++q)
                if (k0 + q < g.nz) gdp[q] = cover_sum_loop<T>(fp, p.partial, comp, i, j, k0 + q);
        } else {
#pragma unroll
            for (int q = 0; q < KZ; ++q)
#pragma unroll
                for (int az = 0; az < 2; ++az)
#pragma unroll
                    for (int ay = 0; ay < 2; ++ay)
#pragma unroll
                        for (int ax = 0; ax < 2; ++ax)
                            if (zsh[q][az] >= 0 && bxy[ay][ax] >= 0) gdp[q] += pv[q][az][ay][ax];
            bool more = false;  // short fused z chunks: covers 3 and 4 (block-uniform)
#pragma unroll
            for (int q = 0; q < KZ; ++q) more |= zsh[q][2] >= 0;
            if (more) {
#pragma unroll
                for (int q = 0; q < KZ; ++q)
#pragma unroll
                    for (int az = 0; az < 2; ++az) {
                        const long long zo = zsh[q][2 + az];
#pragma unroll
                        for (int ay = 0; ay < 2; ++ay)
#pragma unroll
                            for (int ax = 0; ax < 2; ++ax)
                                pv[q][az][ay][ax] = (zo >= 0 && bxy[ay][ax] >= 0) ? __ldcg(p.partial + zo + bxy[ay][ax]) : (T)0;
                    }
#pragma unroll
                for (int q = 0; q < KZ; ++q)
#pragma unroll
                    for (int az = 0; az < 2; ++az)
#pragma unroll
                        for (int ay = 0; ay < 2; ++ay)
#pragma unroll
                            for (int ax = 0; ax < 2; ++ax)
                                if (zsh[q][2 + az] >= 0 && bxy[ay][ax] >= 0) gdp[q] += pv[q][az][ay][ax];
            }
#pragma unroll
            for (int q = 0; q < KZ; ++q)  // more than four z covers: the general loop
                if (zslow[q]) gdp[q] = cover_sum_loop<T>(fp, p.partial, comp, i, j, k0 + q);
        }
    }
    if (mine) {
#pragma unroll
        for (int q = 0; q < KZ; ++q) {
            const int k = k0 + q;
            if (k >= g.nz) break;
            const unsigned idx = ((unsigned)k * g.ny + (unsigned)j) * g.nx + (unsigned)i;
            T gd = p.accumulate ? p.grad[(size_t)comp * m + idx] : (T)0;
            if (p.partial) gd += gdp[q];
            if (yc) {
                // grad S = vol * L^T L u (curvature.py:74-81)
                const int lx = threadIdx.x + 1, ly = threadIdx.y + 1, lz = q + 1;
                const T lc = ls[lz][ly][lx];
                bad |= !isfinite(us[lz + 1][ly + 1][lx + 1]);
                acc += (double)lc * (double)lc;
                T lt = (T)0;
                if (g.nx >= 3) lt = d2t_at<T>(ls[lz][ly][lx - 1], lc, ls[lz][ly][lx + 1], i, g.nx, p.ihx2);
                if (g.ny >= 3) lt = lt + d2t_at<T>(ls[lz][ly - 1][lx], lc, ls[lz][ly + 1][lx], j, g.ny, p.ihy2);
                if (g.nz >= 3) lt = lt + d2t_at<T>(ls[lz - 1][ly][lx], lc, ls[lz + 1][ly][lx], k, g.nz, p.ihz2);
                gd = gd + p.alpha * (p.vol * lt);
            }
            p.grad[(size_t)comp * m + idx] = gd;
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(p.flag, 1);
    if (yc) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (threadIdx.x == 0) red[threadIdx.y] = acc;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < 8; ++w) s += red[w];
            p.spart[bid] = s;
        }
    }
    // last block done: fixed-order totals
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(p.flag + 1, 1) == p.count - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        post_finalize<T>(p, nblk);
    }
}

// ------------------------------------------------------------------ host launchers

void fused_variant_geom(int v, int* ty, int* nt) {
    switch (v) {
        case 1: *ty = V1::TY; *nt = V1::NT; return;
        case 2: *ty = V2::TY; *nt = V2::NT; return;
        case 3: *ty = V3::TY; *nt = V3::NT; return;
        case 4: *ty = V4::TY; *nt = V4::NT; return;
        case 5: *ty = V5::TY; *nt = V5::NT; return;
        case kLeanVariant: *ty = lean::kTYI; *nt = lean::kNT; return;
        case kWsVariant: *ty = kWsTYI; *nt = kWsNT; return;
        default: *ty = V0::TY; *nt = V0::NT; return;
    }
}

int fused_variant_count() { return kNumVariants; }

template <typename T>
size_t fused_smem(int v, int wx, int wy) {
    switch (v) {
        case 1: return smem_bytes_cfg<T, V1>(wx, wy);
        case 2: return smem_bytes_cfg<T, V2>(wx, wy);
        case 3: return smem_bytes_cfg<T, V3>(wx, wy);
        case 4: return smem_bytes_cfg<T, V4>(wx, wy);
        case 5: return smem_bytes_cfg<T, V5>(wx, wy);
        case kLeanVariant: return std::is_same<T, float>::value && wx <= lean::kWXM && wy <= lean::kWYM
                                      ? lean_smem(0, 0) : size_t(1) << 30;
        case kWsVariant: return std::is_same<T, float>::value && wx <= lean::kWXM && wy <= lean::kWYM
                                    ? ws_smem() : size_t(1) << 30;
        default: return smem_bytes_cfg<T, V0>(wx, wy);
    }
}

template <>
int fused_prepare<float>(int v, size_t smem) {
    switch (v) {
        case 1: return march_prepare<float, V1>(smem);
        case 2: return march_prepare<float, V2>(smem);
        case 3: return march_prepare<float, V3>(smem);
        case 4: return march_prepare<float, V4>(smem);
        case 5: return march_prepare<float, V5>(smem);
        case kLeanVariant: return lean_prepare(smem);
        case kWsVariant: return ws_prepare(smem);
        default: return march_prepare<float, V0>(smem);
    }
}

template <>
int fused_prepare<double>(int v, size_t smem) {
    switch (v) {
        case 4: return march_prepare<double, V4>(smem);
        case 5: return march_prepare<double, V5>(smem);
        default: return march_prepare<double, V0>(smem);
    }
}

template <typename T>
static void launch_variant(const FusedArgs<T>& a, cudaStream_t s);

template <>
void launch_variant<float>(const FusedArgs<float>& a, cudaStream_t s) {
    switch (a.fp.variant) {
        case 1: march_launch<float, V1>(a, s); return;
        case 2: march_launch<float, V2>(a, s); return;
        case 3: march_launch<float, V3>(a, s); return;
        case 4: march_launch<float, V4>(a, s); return;
        case 5: march_launch<float, V5>(a, s); return;
        case kLeanVariant: lean_launch(a, *static_cast<const lean::Ctl*>(a.fp.lean_ctl), s); return;
        case kWsVariant: ws_launch(a, *static_cast<const lean::Ctl*>(a.fp.lean_ctl), s); return;
        default: march_launch<float, V0>(a, s); return;
    }
}

template <>
void launch_variant<double>(const FusedArgs<double>& a, cudaStream_t s) {
    switch (a.fp.variant) {
        case 4: march_launch<double, V4>(a, s); return;
        case 5: march_launch<double, V5>(a, s); return;
        default: march_launch<double, V0>(a, s); return;
    }
}

template <typename T>
static PostArgs<T> post_args(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int* flag,
                             T* grad, double* scalars, int part, int nchunk) {
    const double vol = dg.spacing[0] * dg.spacing[1] * dg.spacing[2];
    PostArgs<T> p;
    p.g = make_gridk<T>(dg);
    p.fp = a.fp;
    p.partial = part == 2 ? nullptr : a.partial;
    p.y = part == 1 ? nullptr : a.y;
    p.vol = (T)vol;
    p.alpha = (T)alpha;
    p.grad = grad;
    p.accumulate = part == 2 ? 1 : 0;
    p.dpart = a.dpart;
    p.nd = a.fp.n_cta;
    p.spart = spart;
    p.flag = flag;
    p.half_hbar = a.half_hbar;
    p.half_vol = vol / 2;
    p.dalpha = alpha;
    p.out = scalars;
    p.mode = part;
    p.nchunk = nchunk;
    p.pc0 = 0;
    p.count = (int)(((dg.dims[0] + 31) / 32) * ((dg.dims[1] + 7) / 8)) * 3 * nchunk;
    p.ihx2 = (T)1 / (p.g.hx * p.g.hx);
    p.ihy2 = (T)1 / (p.g.hy * p.g.hy);
    p.ihz2 = (T)1 / (p.g.hz * p.g.hz);
    return p;
}

static int post_chunks(const ngf_grid_t& dg) { return (int)((dg.dims[2] + kPostKZ - 1) / kPostKZ); }

template <typename T>
int fused_eval_launch(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int ns,
                      int* flag, T* grad, double* scalars, cudaStream_t s, cudaEvent_t ev0,
                      cudaEvent_t ev1, int part) {
    // part 0: full evaluation; 1: NGF partial of the level's z-slab (grad <- grad D_slab,
    // scalars <- D_slab); 2: add curvature to an all-reduced (grad D, D) in place
    const int nchunk = post_chunks(dg);
    const dim3 cgrid((dg.dims[0] + 31) / 32, (dg.dims[1] + 7) / 8, 3 * nchunk);
    const int nsb = (int)(cgrid.x * cgrid.y * cgrid.z);
    if (nsb > ns) return NGF_EARG;
    if (part != 2) {
        if (ev0) cudaEventRecord(ev0, s);
        launch_variant<T>(a, s);
        if (ev1) cudaEventRecord(ev1, s);
    }
    const PostArgs<T> p = post_args<T>(a, dg, alpha, spart, flag, grad, scalars, part, nchunk);
    // programmatic dependent launch edges inside conditional graph bodies are opt-in
    // (NGF_GRAPH_PDL=1); a captured evaluation launches k_post plainly by default
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    static const bool graph_pdl = std::getenv("NGF_GRAPH_PDL") != nullptr;
    if (part == 2 || (cap != cudaStreamCaptureStatusNone && !graph_pdl)) {
        NGF_LAUNCH(k_post<T>, cgrid, dim3(32, 8), 0, s, p);
    } else {
        // programmatic dependent launch after the march
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = cgrid;
        cfg.blockDim = dim3(32, 8);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        ::ngf::g_launches.fetch_add(1, std::memory_order_relaxed);
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k_post<T>, p);
        if (e != cudaSuccess) return (int)e;
    }
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int fused_post_range(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int ns, int* flag,
                     T* grad, double* scalars, cudaStream_t s, int pc0, int pc1) {
    const int nchunk = post_chunks(dg);
    if (pc0 < 0 || pc1 > nchunk || pc0 >= pc1) return NGF_EARG;
    const dim3 cgrid((dg.dims[0] + 31) / 32, (dg.dims[1] + 7) / 8, 3 * (pc1 - pc0));
    if ((int)(cgrid.x * cgrid.y) * 3 * nchunk > ns) return NGF_EARG;
    PostArgs<T> p = post_args<T>(a, dg, alpha, spart, flag, grad, scalars, 0, nchunk);
    p.pc0 = pc0;
    NGF_LAUNCH(k_post<T>, cgrid, dim3(32, 8), 0, s, p);
    NGF_CHECK_LAUNCH();
    return 0;
}

void fused_march_launch(const FusedArgs<float>& a, cudaStream_t s) { launch_variant<float>(a, s); }

// packed reference terms (gR / nR, 1 / nR) from the exact ones
template <typename T>
__global__ void k_pack_rt(const T* __restrict__ gR, const T* __restrict__ nR, int64_t n, int64_t first,
                          int64_t last, V4T<T>* __restrict__ out) {
    for (int64_t v = first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < last;
         v += (int64_t)gridDim.x * blockDim.x) {
        const T inv = (T)1 / nR[v];
        V4T<T> r;
        r.x = gR[v] * inv;
        r.y = gR[n + v] * inv;
        r.z = gR[2 * n + v] * inv;
        r.w = inv;
        out[v] = r;
    }
}

// voxels [first, last) of n (last < 0: all)
template <typename T>
int pack_rt(const T* gR, const T* nR, int64_t n, void* out, cudaStream_t s, int64_t first, int64_t last) {
    if (last < 0) last = n;
    NGF_LAUNCH(k_pack_rt<T>, blocks_for(last - first, 256), 256, 0, s, gR, nR, n, first, last, (V4T<T>*)out);
    NGF_CHECK_LAUNCH();
    return 0;
}


template int fused_eval_launch<float>(const FusedArgs<float>&, const ngf_grid_t&, double, double*, int,
                                      int*, float*, double*, cudaStream_t, cudaEvent_t, cudaEvent_t,
                                      int);
template int fused_eval_launch<double>(const FusedArgs<double>&, const ngf_grid_t&, double, double*,
                                       int, int*, double*, double*, cudaStream_t, cudaEvent_t,
                                       cudaEvent_t, int);
template int fused_post_range<float>(const FusedArgs<float>&, const ngf_grid_t&, double, double*, int, int*,
                                     float*, double*, cudaStream_t, int, int);
template size_t fused_smem<float>(int, int, int);
template size_t fused_smem<double>(int, int, int);
template int pack_rt<float>(const float*, const float*, int64_t, void*, cudaStream_t, int64_t, int64_t);
template int pack_rt<double>(const double*, const double*, int64_t, void*, cudaStream_t, int64_t, int64_t);

}  // namespace ngf
