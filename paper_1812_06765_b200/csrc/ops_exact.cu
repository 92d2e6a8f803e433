// Standalone operators, bit-exact re-statements of the reference (sm_100a).
//
// This translation unit is compiled with --fmad=false and IEEE div/sqrt, so each
// C++ arithmetic expression below is one correctly rounded operation in the
// order written -- the same order numpy evaluates the reference expressions.
// Signed zeros are reproduced too (accumulators start at +0 like np.zeros).
//
// These kernels are the parity path (mode 1 of ngf_level_eval) and the
// standalone operator API; the performance path is eval_fused.cu.

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ops_exact.cuh"

namespace ngf {

// ------------------------------------------------------------------ P (transfer.py:117-148)

template <typename T>
__device__ __forceinline__ T lerp_ref(T a0, T a1, T w) {
    // a0 * (1 - w) + a1 * w  (transfer.py:126)
    return a0 * ((T)1 - w) + a1 * w;
}

template <typename T>
__global__ void k_apply_P(AxisDev ax, AxisDev ay, AxisDev az, const T* __restrict__ y,
                          T* __restrict__ out) {
    const int nx = ax.ni, ny = ay.ni, nz = az.ni;
    const int ndx = ax.nd, ndy = ay.nd, ndz = az.nd;
    const int64_t n = (int64_t)nx * ny * nz;
    const int64_t m = (int64_t)ndx * ndy * ndz;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(v % nx);
        const int j = (int)((v / nx) % ny);
        const int k = (int)(v / ((int64_t)nx * ny));
        const int x0 = ax.i0[i], x1 = min(x0 + 1, ndx - 1);
        const int y0 = ay.i0[j], y1 = min(y0 + 1, ndy - 1);
        const int z0 = az.i0[k], z1 = min(z0 + 1, ndz - 1);
        const T wx = w1_of<T>(ax)[i], wy = w1_of<T>(ay)[j], wz = w1_of<T>(az)[k];
        for (int c = 0; c < 3; ++c) {
            const T* yc = y + c * m;
            T Y[2];
#pragma unroll
            for (int dz = 0; dz < 2; ++dz) {
                const int zz = dz ? z1 : z0;
                const T* p0 = yc + ((int64_t)zz * ndy + y0) * ndx;
                const T* p1 = yc + ((int64_t)zz * ndy + y1) * ndx;
                T X0 = lerp_ref(p0[x0], p0[x1], wx);
                T X1 = lerp_ref(p1[x0], p1[x1], wx);
                Y[dz] = lerp_ref(X0, X1, wy);
            }
            out[c * n + v] = lerp_ref(Y[0], Y[1], wz);
        }
    }
}

template <typename T>
int apply_P_impl(const ngf_plan_t* p, const T* y, T* out, cudaStream_t s) {
    if (int rc = plan_upload(const_cast<ngf_plan_t*>(p))) return rc;
    int64_t n = grid_n(p->img_grid);
    NGF_LAUNCH(k_apply_P<T>, blocks_for(n, 256), 256, 0, s, p->axes[0], p->axes[1], p->axes[2], y,
               out);
    NGF_CHECK_LAUNCH();
    return 0;
}

// ------------------------------------------------------------------ P^T gather (transfer.py:151-192)

// Stage A: tmp[c][k][dy][dx] = sum_jy Wy[dy,jy] * (sum_jx r[c][k][ys+jy][xs+jx] * Wx[dx,jx])
template <typename T>
__global__ void k_pt_xy(AxisDev ax, AxisDev ay, int nz, const T* __restrict__ r,
                        T* __restrict__ tmp) {
    const int nx = ax.ni, ny = ay.ni, ndx = ax.nd, ndy = ay.nd;
    const int wxn = ax.width, wyn = ay.width;
    const int64_t tot = (int64_t)3 * nz * ndy * ndx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < tot;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int dx = (int)(v % ndx);
        const int dy = (int)((v / ndx) % ndy);
        const int64_t ck = v / ((int64_t)ndx * ndy);  // c * nz + k
        const T* row0 = r + ck * ((int64_t)nx * ny);
        const int xs = ax.start[dx], ys = ay.start[dy];
        const T* Wx = wts_of<T>(ax) + (int64_t)dx * wxn;
        const T* Wy = wts_of<T>(ay) + (int64_t)dy * wyn;
        T acc_y = 0;
        for (int jy = 0; jy < wyn; ++jy) {
            const int yy = min(ys + jy, ny - 1);
            const T* row = row0 + (int64_t)yy * nx;
            T acc_x = row[min(xs, nx - 1)] * Wx[0];
            for (int jx = 1; jx < wxn; ++jx) acc_x = acc_x + row[min(xs + jx, nx - 1)] * Wx[jx];
            T term = acc_x * Wy[jy];
            acc_y = jy == 0 ? term : acc_y + term;
        }
        tmp[v] = acc_y;
    }
}

// Stage B: out[c][dz][dy][dx] = sum_jz tmp[c][zs+jz][dy][dx] * Wz[dz,jz]
template <typename T>
__global__ void k_pt_z(AxisDev az, int ndy, int ndx, const T* __restrict__ tmp,
                       T* __restrict__ out) {
    const int nz = az.ni, ndz = az.nd, wzn = az.width;
    const int64_t plane = (int64_t)ndy * ndx;
    const int64_t tot = (int64_t)3 * ndz * plane;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < tot;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xy = v % plane;
        const int dz = (int)((v / plane) % ndz);
        const int c = (int)(v / (plane * ndz));
        const T* base = tmp + (int64_t)c * nz * plane + xy;
        const T* Wz = wts_of<T>(az) + (int64_t)dz * wzn;
        const int zs = az.start[dz];
        T acc = base[(int64_t)min(zs, nz - 1) * plane] * Wz[0];
        for (int jz = 1; jz < wzn; ++jz) acc = acc + base[(int64_t)min(zs + jz, nz - 1) * plane] * Wz[jz];
        out[v] = acc;
    }
}

template <typename T>
int apply_Pt_impl(const ngf_plan_t* p, const T* r, T* out, cudaStream_t s) {
    if (int rc = plan_upload(const_cast<ngf_plan_t*>(p))) return rc;
    const int nz = p->n_img[2], ndy = p->n_def[1], ndx = p->n_def[0], ndz = p->n_def[2];
    T* tmp = (T*)p->d_tmp;
    int64_t ta = (int64_t)3 * nz * ndy * ndx;
    NGF_LAUNCH(k_pt_xy<T>, blocks_for(ta, 256), 256, 0, s, p->axes[0], p->axes[1], nz, r, tmp);
    int64_t tb = (int64_t)3 * ndz * ndy * ndx;
    NGF_LAUNCH(k_pt_z<T>, blocks_for(tb, 256), 256, 0, s, p->axes[2], ndy, ndx, tmp, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

// ------------------------------------------------------------------ P^T scatter / red-black
// The reference's two other P^T variants (transfer.py:199-256): the image slices are
// reduced in x then y exactly like the gather (k_pt_xy, `_reduce_slice_xy`), then each
// slice k is pushed onto def planes i0z[k] and i0z[k]+1 with w1 = dtype(w1z[k]),
// w0 = 1 - w1 (working dtype), `out += w * sl` (product then sum, no contraction).

// scatter: one thread per reduced slice value, float atomics (order is not fixed:
// equal to the gather up to floating-point reassociation, like the reference's
// lock-based scatter, transfer.py:199-222)
template <typename T>
__global__ void k_pt_z_scatter(AxisDev az, int ndy, int ndx, const T* __restrict__ tmp, T* __restrict__ out) {
    const int nz = az.ni, ndz = az.nd;
    const int64_t plane = (int64_t)ndy * ndx;
    const int64_t tot = (int64_t)3 * nz * plane;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < tot;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xy = v % plane;
        const int k = (int)((v / plane) % nz);
        const int c = (int)(v / (plane * nz));
        const T val = tmp[v];
        const T w1 = w1_of<T>(az)[k];
        const T w0 = (T)1 - w1;
        T* o = out + ((int64_t)c * ndz + az.i0[k]) * plane + xy;
        atomicAdd(o, w0 * val);
        if (w1 != (T)0) atomicAdd(o + plane, w1 * val);
    }
}

// red-black: slices grouped by their lower def plane d0 (a contiguous k range, i0z is
// non-decreasing); one launch per parity of d0, one thread per (component, group,
// def column) adding the group's slices in ascending k.  Groups of one colour write
// disjoint planes, so every output receives its terms in the reference's order
// (transfer.py:225-256): bit-identical to the reference.
template <typename T>
__global__ void k_pt_z_redblack(AxisDev az, int ndy, int ndx, int parity, const T* __restrict__ tmp,
                                T* __restrict__ out) {
    const int nz = az.ni, ndz = az.nd;
    const int ng = (ndz - parity + 1) / 2;  // candidate groups d0 = parity, parity + 2, ...
    const int64_t plane = (int64_t)ndy * ndx;
    const int64_t tot = (int64_t)3 * ng * plane;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < tot;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t xy = v % plane;
        const int gi = (int)((v / plane) % ng);
        const int c = (int)(v / (plane * ng));
        const int d0 = parity + 2 * gi;
        // slices with i0z[k] == d0: [lo, hi) by binary search
        int lo = 0, hi = nz;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (az.i0[mid] < d0) lo = mid + 1; else hi = mid;
        }
        int k1 = lo, e = nz;
        while (k1 < e) {
            const int mid = (k1 + e) >> 1;
            if (az.i0[mid] <= d0) k1 = mid + 1; else e = mid;
        }
        if (lo == k1) continue;  // empty group
        T* o0 = out + ((int64_t)c * ndz + d0) * plane + xy;
        const T* src = tmp + (int64_t)c * nz * plane + xy;
        for (int k = lo; k < k1; ++k) {
            const T val = src[(int64_t)k * plane];
            const T w1 = w1_of<T>(az)[k];
            const T w0 = (T)1 - w1;
            o0[0] = o0[0] + w0 * val;
            if (w1 != (T)0) o0[plane] = o0[plane] + w1 * val;
        }
    }
}

template <typename T>
int apply_Pt_variant_impl(const ngf_plan_t* p, int variant, const T* r, T* out, cudaStream_t s) {
    if (variant == 0) return apply_Pt_impl<T>(p, r, out, s);
    if (variant != 1 && variant != 2) return NGF_EARG;
    if (int rc = plan_upload(const_cast<ngf_plan_t*>(p))) return rc;
    const int nz = p->n_img[2], ndy = p->n_def[1], ndx = p->n_def[0], ndz = p->n_def[2];
    T* tmp = (T*)p->d_tmp;
    const int64_t ta = (int64_t)3 * nz * ndy * ndx;
    NGF_LAUNCH(k_pt_xy<T>, blocks_for(ta, 256), 256, 0, s, p->axes[0], p->axes[1], nz, r, tmp);
    NGF_CUDA(cudaMemsetAsync(out, 0, (size_t)3 * ndz * ndy * ndx * sizeof(T), s));
    if (variant == 1) {
        NGF_LAUNCH(k_pt_z_scatter<T>, blocks_for(ta, 256), 256, 0, s, p->axes[2], ndy, ndx, tmp, out);
    } else {
        for (int parity = 0; parity < 2; ++parity) {
            const int64_t tb = (int64_t)3 * ((ndz - parity + 1) / 2) * ndy * ndx;
            if (tb > 0)
                NGF_LAUNCH(k_pt_z_redblack<T>, blocks_for(tb, 256), 256, 0, s, p->axes[2], ndy, ndx, parity,
                           tmp, out);
        }
    }
    NGF_CHECK_LAUNCH();
    return 0;
}

// ------------------------------------------------------------------ warp (warp.py:26-127)

template <typename T>
struct CellCoords {
    bool inside;
    int i0[3];
    T f[3];
};

template <typename T>
__device__ __forceinline__ CellCoords<T> cell_coords(const GridK<T>& g, T px, T py, T pz) {
    // warp.py:32-53: t = (p - origin) / h in the working dtype; inside test on t;
    // i0 = clip(floor(t), 0, max(n-2, 0)); f = clip(t - i0, 0, 1)
    CellCoords<T> c;
    const T p[3] = {px, py, pz};
    const T o[3] = {g.ox, g.oy, g.oz};
    const T h[3] = {g.hx, g.hy, g.hz};
    const int n[3] = {g.nx, g.ny, g.nz};
    c.inside = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        T t = (p[a] - o[a]) / h[a];
        c.inside = c.inside && (t >= (T)0) && (t <= (T)(n[a] - 1));
        T fl = floor(t);
        int hi = max(n[a] - 2, 0);
        int lo;
        if (!(fl >= (T)0))
            lo = 0;  // also NaN
        else if (fl > (T)hi)
            lo = hi;
        else
            lo = (int)fl;
        c.i0[a] = lo;
        // t - i0 in f64 then cast (numpy promotes f32 - int64 to f64)
        double fr = (double)t - (double)lo;
        fr = fr < 0.0 ? 0.0 : (fr > 1.0 ? 1.0 : fr);
        c.f[a] = (T)fr;
    }
    return c;
}

template <typename T>
__device__ __forceinline__ T corner(const T* __restrict__ Tv, const GridK<T>& g,
                                    const CellCoords<T>& c, int dx, int dy, int dz) {
    const int ix = min(c.i0[0] + dx, g.nx - 1);
    const int iy = min(c.i0[1] + dy, g.ny - 1);
    const int iz = min(c.i0[2] + dz, g.nz - 1);
    return Tv[((int64_t)iz * g.ny + iy) * g.nx + ix];
}

template <typename T>
__global__ void k_warp(GridK<T> g, const T* __restrict__ Tv, const T* __restrict__ yhat, int64_t n,
                       T* __restrict__ W, uint8_t* __restrict__ mask) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        CellCoords<T> c = cell_coords(g, yhat[v], yhat[n + v], yhat[2 * n + v]);
        T acc = 0;
#pragma unroll
        for (int dz = 0; dz < 2; ++dz) {
            const T wz = dz ? c.f[2] : (T)1 - c.f[2];
#pragma unroll
            for (int dy = 0; dy < 2; ++dy) {
                const T wy = dy ? c.f[1] : (T)1 - c.f[1];
#pragma unroll
                for (int dx = 0; dx < 2; ++dx) {
                    const T wx = dx ? c.f[0] : (T)1 - c.f[0];
                    acc = acc + corner(Tv, g, c, dx, dy, dz) * (wx * wy * wz);
                }
            }
        }
        W[v] = c.inside ? acc : (T)0;
        if (mask) mask[v] = c.inside ? 1 : 0;
    }
}

template <typename T>
__global__ void k_warp_jt(GridK<T> g, const T* __restrict__ Tv, const T* __restrict__ yhat,
                          const T* __restrict__ s, int64_t n, T* __restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        CellCoords<T> c = cell_coords(g, yhat[v], yhat[n + v], yhat[2 * n + v]);
        T gx = 0, gy = 0, gz = 0;
#pragma unroll
        for (int dz = 0; dz < 2; ++dz) {
            const T wz = dz ? c.f[2] : (T)1 - c.f[2];
            const T sz = dz ? (T)1 : (T)-1;
#pragma unroll
            for (int dy = 0; dy < 2; ++dy) {
                const T wy = dy ? c.f[1] : (T)1 - c.f[1];
                const T sy = dy ? (T)1 : (T)-1;
#pragma unroll
                for (int dx = 0; dx < 2; ++dx) {
                    const T wx = dx ? c.f[0] : (T)1 - c.f[0];
                    const T sx = dx ? (T)1 : (T)-1;
                    const T cv = corner(Tv, g, c, dx, dy, dz);
                    gx = gx + cv * (sx * wy * wz);
                    gy = gy + cv * (wx * sy * wz);
                    gz = gz + cv * (wx * wy * sz);
                }
            }
        }
        const T sv = s[v];
        // warp.py:123: scale = s / h if dims > 1 else 0.0
        const T kx = g.nx > 1 ? sv / g.hx : (T)0;
        const T ky = g.ny > 1 ? sv / g.hy : (T)0;
        const T kz = g.nz > 1 ? sv / g.hz : (T)0;
        out[v] = c.inside ? gx * kx : (T)0;
        out[n + v] = c.inside ? gy * ky : (T)0;
        out[2 * n + v] = c.inside ? gz * kz : (T)0;
    }
}

// ------------------------------------------------------------------ G, G^T (warp.py:130-184)

template <typename T>
__device__ __forceinline__ T fd_axis(const T* v, int64_t idx, int i, int n, int64_t stride, T h) {
    // warp.py:130-143
    if (n < 2) return (T)0;
    if (i == 0) return (v[idx + stride] - v[idx]) / h;
    if (i == n - 1) return (v[idx] - v[idx - stride]) / h;
    return (v[idx + stride] - v[idx - stride]) / ((T)2 * h);
}

template <typename T>
__global__ void k_gradient(GridK<T> g, const T* __restrict__ v, T* __restrict__ out) {
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        out[idx] = fd_axis(v, idx, i, g.nx, 1, g.hx);
        out[n + idx] = fd_axis(v, idx, j, g.ny, sy, g.hy);
        out[2 * n + idx] = fd_axis(v, idx, k, g.nz, sz, g.hz);
    }
}

template <typename T>
__device__ __forceinline__ T fd_t_axis(const T* w, int64_t idx, int i, int n, int64_t stride, T h) {
    // warp.py:159-176, same update sequence as the numpy slices, starting from +0
    T o = 0;
    if (n < 2) return o;
    if (i == 0) o = o + (-w[idx] / h);
    if (i == 1) o = o + w[idx - stride] / h;
    if (i == n - 2) o = o + (-w[idx + stride] / h);
    if (i == n - 1) o = o + w[idx] / h;
    if (n > 2) {
        const T h2 = (T)2 * h;
        if (i <= n - 3) o = o + (-(w[idx + stride] / h2));
        if (i >= 2) o = o + w[idx - stride] / h2;
    }
    return o;
}

template <typename T>
__global__ void k_gradient_t(GridK<T> g, const T* __restrict__ w, T* __restrict__ out) {
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        T acc = 0;
        acc = acc + fd_t_axis(w, idx, i, g.nx, 1, g.hx);
        acc = acc + fd_t_axis(w + n, idx, j, g.ny, sy, g.hy);
        acc = acc + fd_t_axis(w + 2 * n, idx, k, g.nz, sz, g.hz);
        out[idx] = acc;
    }
}

// ------------------------------------------------------------------ NGF terms (ngf.py:60-114)

template <typename T>
__global__ void k_ref_terms(GridK<T> g, const T* __restrict__ R, T rho, T* __restrict__ gR,
                            T* __restrict__ nR, int64_t first, int64_t last) {
    // voxels [first, last) (a z-slab of planes for the config-5 decomposition; R is read on
    // the neighbouring planes as well, so the slab needs no halo exchange)
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const T rho2 = rho * rho;
    for (int64_t idx = first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < last;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        const T ax = fd_axis(R, idx, i, g.nx, 1, g.hx);
        const T ay = fd_axis(R, idx, j, g.ny, sy, g.hy);
        const T az = fd_axis(R, idx, k, g.nz, sz, g.hz);
        gR[idx] = ax;
        gR[n + idx] = ay;
        gR[2 * n + idx] = az;
        T sq = 0;
        sq = sq + ax * ax;
        sq = sq + ay * ay;
        sq = sq + az * az;
        nR[idx] = sqrt(sq + rho2);
    }
}

template <typename T>
__global__ void k_ngf_terms(GridK<T> g, const T* __restrict__ W, const T* __restrict__ gR,
                            const T* __restrict__ nR, T tau2, T taurho, T neg_hbar,
                            T* __restrict__ terms, T* __restrict__ q) {
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        const T t0 = fd_axis(W, idx, i, g.nx, 1, g.hx);
        const T t1 = fd_axis(W, idx, j, g.ny, sy, g.hy);
        const T t2 = fd_axis(W, idx, k, g.nz, sz, g.hz);
        const T r0 = gR[idx], r1 = gR[n + idx], r2 = gR[2 * n + idx];
        const T nr = nR[idx];
        // _ratio_terms (ngf.py:70-80)
        T dot = 0, sq = 0;
        dot = dot + t0 * r0;
        sq = sq + t0 * t0;
        dot = dot + t1 * r1;
        sq = sq + t1 * t1;
        dot = dot + t2 * r2;
        sq = sq + t2 * t2;
        const T nT = sqrt(sq + tau2);
        const T r = (dot + taurho) / (nT * nr);
        if (terms) terms[idx] = (T)1 - r * r;  // ngf.py:89
        if (q) {
            // ngf.py:106-112
            const T coef = neg_hbar * r;
            const T inv_prod = (T)1 / (nT * nr);
            const T inv_nt2 = (T)1 / (nT * nT);
            q[idx] = coef * (r0 * inv_prod - r * t0 * inv_nt2);
            q[n + idx] = coef * (r1 * inv_prod - r * t1 * inv_nt2);
            q[2 * n + idx] = coef * (r2 * inv_prod - r * t2 * inv_nt2);
        }
    }
}

// ------------------------------------------------------------------ numpy pairwise sum

// Leaf of numpy's pairwise summation (n <= 128): 8 strided accumulators,
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the remainder in order.
template <typename T>
__device__ T pairwise_leaf(const T* a, int64_t n) {
    if (n < 8) {
        T res = 0;
        for (int64_t i = 0; i < n; ++i) res = res + a[i];
        return res;
    }
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    }
    T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i];
    return res;
}

// One pass of the pairwise tree: node v combines children (left, right) or, for
// a leaf, sums its segment.  Nodes of one height are independent.
struct PwNode {
    int64_t off, len;  // leaf: segment; internal: unused
    int32_t left, right;  // child node ids, -1 for leaf
};

template <typename T>
__global__ void k_pairwise_level(const T* __restrict__ x, const PwNode* __restrict__ nodes,
                                 const int32_t* __restrict__ ids, int count, T* __restrict__ vals) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
        const int id = ids[t];
        const PwNode nd = nodes[id];
        if (nd.left < 0)
            vals[id] = pairwise_leaf(x + nd.off, nd.len);
        else
            vals[id] = vals[nd.left] + vals[nd.right];
    }
}

template <typename T>
__global__ void k_store_root(const T* vals, int root, double* out, int mode, double scale) {
    // mode 0: raw sum; mode 1: value = scale * sum with the dtype rounding of
    // `python_float * numpy_scalar` (NEP 50: the python float is cast to T).
    T s = vals[root];
    if (mode == 0)
        *out = (double)s;
    else
        *out = (double)((T)scale * s);
}

struct PwProgram {
    std::vector<PwNode> nodes;
    std::vector<std::vector<int32_t>> levels;  // node ids per height
    int root;
    void* d_nodes = nullptr;
    void* d_ids = nullptr;
    std::vector<size_t> level_off;
    void* d_vals = nullptr;
};

static int build_pw(int64_t off, int64_t n, PwProgram& P, int& height) {
    PwNode nd{off, n, -1, -1};
    if (n <= 128) {
        P.nodes.push_back(nd);
        height = 0;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        int hl, hr;
        int l = build_pw(off, n2, P, hl);
        int r = build_pw(off + n2, n - n2, P, hr);
        nd.left = l;
        nd.right = r;
        P.nodes.push_back(nd);
        height = 1 + (hl > hr ? hl : hr);
    }
    int id = (int)P.nodes.size() - 1;
    if ((int)P.levels.size() <= height) P.levels.resize(height + 1);
    P.levels[height].push_back(id);
    return id;
}

static std::mutex g_pw_mu;
static std::map<std::pair<int64_t, cudaStream_t>, PwProgram*> g_pw_cache;

static PwProgram* get_pw(int64_t n, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_pw_mu);
    auto it = g_pw_cache.find({n, s});
    if (it != g_pw_cache.end()) return it->second;
    PwProgram* P = new PwProgram();
    int h;
    P->root = build_pw(0, n, *P, h);
    std::vector<int32_t> flat;
    for (auto& lv : P->levels) {
        P->level_off.push_back(flat.size());
        flat.insert(flat.end(), lv.begin(), lv.end());
    }
    if (cudaMalloc(&P->d_nodes, P->nodes.size() * sizeof(PwNode)) != cudaSuccess ||
        cudaMalloc(&P->d_ids, flat.size() * 4) != cudaSuccess ||
        cudaMalloc(&P->d_vals, P->nodes.size() * 8) != cudaSuccess) {
        delete P;
        return nullptr;
    }
    if (upload_blocking(P->d_nodes, P->nodes.data(), P->nodes.size() * sizeof(PwNode)) ||
        upload_blocking(P->d_ids, flat.data(), flat.size() * 4)) {
        delete P;
        return nullptr;
    }
    g_pw_cache[{n, s}] = P;
    return P;
}

// The cached program (and its value buffer) belongs to one (n, stream): calls on one
// stream are ordered, calls on different streams use different buffers.
template <typename T>
int pairwise_sum_impl(const T* x, int64_t n, double* out, int mode, double scale, cudaStream_t s) {
    if (n <= 0) {
        double z = 0.0;
        NGF_CUDA(cudaMemcpyAsync(out, &z, 8, cudaMemcpyHostToDevice, s));
        return 0;
    }
    PwProgram* P = get_pw(n, s);
    if (!P) return NGF_ENOMEM;
    for (size_t h = 0; h < P->levels.size(); ++h) {
        int cnt = (int)P->levels[h].size();
        const int32_t* ids = (const int32_t*)P->d_ids + P->level_off[h];
        NGF_LAUNCH(k_pairwise_level<T>, blocks_for(cnt, 128), 128, 0, s, x,
                   (const PwNode*)P->d_nodes, ids, cnt, (T*)P->d_vals);
    }
    NGF_LAUNCH(k_store_root<T>, 1, 1, 0, s, (const T*)P->d_vals, P->root, out, mode, scale);
    NGF_CHECK_LAUNCH();
    return 0;
}

// ------------------------------------------------------------------ curvature (curvature.py:20-81)

template <typename T>
__device__ __forceinline__ T d2_axis(const T* v, int64_t idx, int i, int n, int64_t stride, T h2) {
    // (v[i+1] - 2*v[i] + v[i-1]) / h2 on interior rows, 0 at faces / n < 3
    if (n < 3 || i == 0 || i == n - 1) return (T)0;
    return (v[idx + stride] - (T)2 * v[idx] + v[idx - stride]) / h2;
}

template <typename T>
__device__ __forceinline__ T d2t_axis(const T* w, int64_t idx, int i, int n, int64_t stride, T h2) {
    // rr[:-2] += mid; rr[1:-1] -= 2*mid; rr[2:] += mid with mid = w[1:-1]/h2
    T o = 0;
    if (n < 3) return o;
    if (i <= n - 3) o = o + w[idx + stride] / h2;
    if (i >= 1 && i <= n - 2) o = o - (T)2 * (w[idx] / h2);
    if (i >= 2) o = o + w[idx - stride] / h2;
    return o;
}

template <typename T>
__global__ void k_laplacian(GridK<T> g, const T* __restrict__ u, T* __restrict__ out, int ncomp) {
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const T hx2 = g.hx * g.hx, hy2 = g.hy * g.hy, hz2 = g.hz * g.hz;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ncomp;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = t % n;
        const T* uc = u + (t / n) * n;
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        T acc = 0;
        acc = acc + d2_axis(uc, idx, i, g.nx, 1, hx2);
        acc = acc + d2_axis(uc, idx, j, g.ny, sy, hy2);
        acc = acc + d2_axis(uc, idx, k, g.nz, sz, hz2);
        out[t] = acc;
    }
}

template <typename T>
__global__ void k_laplacian_t(GridK<T> g, const T* __restrict__ w, T* __restrict__ out, int ncomp,
                              T scale, int use_scale, const T* __restrict__ add, T add_scale,
                              T* __restrict__ sq_out) {
    const int64_t n = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const T hx2 = g.hx * g.hx, hy2 = g.hy * g.hy, hz2 = g.hz * g.hz;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ncomp;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = t % n;
        const T* wc = w + (t / n) * n;
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        T acc = 0;
        acc = acc + d2t_axis(wc, idx, i, g.nx, 1, hx2);
        acc = acc + d2t_axis(wc, idx, j, g.ny, sy, hy2);
        acc = acc + d2t_axis(wc, idx, k, g.nz, sz, hz2);
        if (use_scale) acc = scale * acc;
        if (add) acc = add[t] + add_scale * acc;  // objective.py:50: grad_D + f(alpha) * grad_S
        out[t] = acc;
        (void)sq_out;
    }
}

// u = y - identity (geometry.py:148-163): identity computed in f64 then cast
template <typename T>
__global__ void k_displacement(GridK<T> g, const T* __restrict__ y, T* __restrict__ u) {
    const int64_t n = g.n();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(t / n);
        const int64_t idx = t % n;
        int i;
        double o, h;
        if (c == 0) {
            i = (int)(idx % g.nx);
            o = g.dox;
            h = g.dhx;
        } else if (c == 1) {
            i = (int)((idx / g.nx) % g.ny);
            o = g.doy;
            h = g.dhy;
        } else {
            i = (int)(idx / ((int64_t)g.nx * g.ny));
            o = g.doz;
            h = g.dhz;
        }
        const T id = (T)(o + h * (double)i);
        u[t] = y[t] - id;
    }
}

template <typename T>
__global__ void k_square(const T* __restrict__ a, T* __restrict__ out, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        out[t] = a[t] * a[t];
}

// S total: tot = T(0); tot = tot + sum_c (per component pairwise sums), then
// S = float(vol/2 * tot) (curvature.py:66-71)
template <typename T>
__global__ void k_curv_total(const double* sums, double half_vol, double* out) {
    T tot = 0;
    for (int c = 0; c < 3; ++c) tot = tot + (T)sums[c];
    *out = (double)((T)half_vol * tot);
}

// ------------------------------------------------------------------ pyramid (multilevel.py:100-121)

template <typename T>
__global__ void k_downsample(int nx, int ny, int nz, const T* __restrict__ in, T* __restrict__ out) {
    // per axis z, y, x in turn: (a + b) / count (count 1 at an odd tail)
    const int mx = nx > 1 ? (nx + 1) / 2 : 1;
    const int my = ny > 1 ? (ny + 1) / 2 : 1;
    const int mz = nz > 1 ? (nz + 1) / 2 : 1;
    const int64_t m = (int64_t)mx * my * mz;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(v % mx);
        const int j = (int)((v / mx) % my);
        const int k = (int)(v / ((int64_t)mx * my));
        const int x0 = nx > 1 ? 2 * i : 0, cx = nx > 1 ? min(2, nx - x0) : 1;
        const int y0 = ny > 1 ? 2 * j : 0, cy = ny > 1 ? min(2, ny - y0) : 1;
        const int z0 = nz > 1 ? 2 * k : 0, cz = nz > 1 ? min(2, nz - z0) : 1;
        // reference order: z-stage, then y-stage, then x-stage
        T Xv[2];
        for (int dx = 0; dx < cx; ++dx) {
            T Ys[2];
            for (int dy = 0; dy < cy; ++dy) {
                const T* p = in + ((int64_t)z0 * ny + (y0 + dy)) * nx + (x0 + dx);
                T zs = p[0];
                if (nz > 1) {
                    if (cz == 2) zs = zs + p[(int64_t)nx * ny];
                    zs = zs / (T)cz;
                }
                Ys[dy] = zs;
            }
            T ys = Ys[0];
            if (ny > 1) {
                if (cy == 2) ys = ys + Ys[1];
                ys = ys / (T)cy;
            }
            Xv[dx] = ys;
        }
        T xs = Xv[0];
        if (nx > 1) {
            if (cx == 2) xs = xs + Xv[1];
            xs = xs / (T)cx;
        }
        out[v] = xs;
    }
}

// ------------------------------------------------------------------ prolongation (multilevel.py:163-176)

template <typename T>
__global__ void k_prolong(AxisDev ax, AxisDev ay, AxisDev az, GridK<T> gc, GridK<T> gf,
                          const T* __restrict__ yc, T* __restrict__ yf) {
    const int nx = ax.ni, ny = ay.ni, nz = az.ni;
    const int ndx = ax.nd, ndy = ay.nd, ndz = az.nd;
    const int64_t n = (int64_t)nx * ny * nz;
    const int64_t m = (int64_t)ndx * ndy * ndz;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(v % nx);
        const int j = (int)((v / nx) % ny);
        const int k = (int)(v / ((int64_t)nx * ny));
        const int x0 = ax.i0[i], x1 = min(x0 + 1, ndx - 1);
        const int y0 = ay.i0[j], y1 = min(y0 + 1, ndy - 1);
        const int z0 = az.i0[k], z1 = min(z0 + 1, ndz - 1);
        const T wx = w1_of<T>(ax)[i], wy = w1_of<T>(ay)[j], wz = w1_of<T>(az)[k];
        // coarse identity values (f64 centers cast to T)
        const T idcx0 = (T)(gc.dox + gc.dhx * (double)x0), idcx1 = (T)(gc.dox + gc.dhx * (double)x1);
        const T idcy0 = (T)(gc.doy + gc.dhy * (double)y0), idcy1 = (T)(gc.doy + gc.dhy * (double)y1);
        const T idcz0 = (T)(gc.doz + gc.dhz * (double)z0), idcz1 = (T)(gc.doz + gc.dhz * (double)z1);
        const T idf[3] = {(T)(gf.dox + gf.dhx * (double)i), (T)(gf.doy + gf.dhy * (double)j),
                          (T)(gf.doz + gf.dhz * (double)k)};
        for (int c = 0; c < 3; ++c) {
            const T* ycc = yc + c * m;
            T Y[2];
#pragma unroll
            for (int dz = 0; dz < 2; ++dz) {
                const int zz = dz ? z1 : z0;
                T X[2];
#pragma unroll
                for (int dy = 0; dy < 2; ++dy) {
                    const int yy = dy ? y1 : y0;
                    const T* p = ycc + ((int64_t)zz * ndy + yy) * ndx;
                    T a0 = p[x0], a1 = p[x1];
                    // u = y - id(coarse) for this component
                    T i0v, i1v;
                    if (c == 0) {
                        i0v = idcx0;
                        i1v = idcx1;
                    } else if (c == 1) {
                        i0v = i1v = dy ? idcy1 : idcy0;
                    } else {
                        i0v = i1v = dz ? idcz1 : idcz0;
                    }
                    a0 = a0 - i0v;
                    a1 = a1 - i1v;
                    X[dy] = lerp_ref(a0, a1, wx);
                }
                Y[dz] = lerp_ref(X[0], X[1], wy);
            }
            const T u = lerp_ref(Y[0], Y[1], wz);
            yf[c * n + v] = idf[c] + u;
        }
    }
}

// ------------------------------------------------------------------ host entry points

template <typename T>
int warp_impl(const ngf_grid_t* tg, const T* Tv, const T* yhat, int64_t n, T* W, uint8_t* mask,
              cudaStream_t s) {
    NGF_LAUNCH(k_warp<T>, blocks_for(n, 256), 256, 0, s, make_gridk<T>(*tg), Tv, yhat, n, W, mask);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int warp_jt_impl(const ngf_grid_t* tg, const T* Tv, const T* yhat, const T* sv, int64_t n, T* out,
                 cudaStream_t s) {
    NGF_LAUNCH(k_warp_jt<T>, blocks_for(n, 256), 256, 0, s, make_gridk<T>(*tg), Tv, yhat, sv, n,
               out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int gradient_impl(const ngf_grid_t* g, const T* v, T* out, cudaStream_t s) {
    NGF_LAUNCH(k_gradient<T>, blocks_for(grid_n(*g), 256), 256, 0, s, make_gridk<T>(*g), v, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int gradient_t_impl(const ngf_grid_t* g, const T* w, T* out, cudaStream_t s) {
    NGF_LAUNCH(k_gradient_t<T>, blocks_for(grid_n(*g), 256), 256, 0, s, make_gridk<T>(*g), w, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int ref_terms_impl(const ngf_grid_t* g, const T* R, double rho, T* gR, T* nR, cudaStream_t s,
                   int64_t zlo, int64_t zhi) {
    const int64_t plane = g->dims[0] * g->dims[1];
    if (zhi < 0) zhi = g->dims[2];
    const int64_t first = zlo * plane, last = zhi * plane;
    NGF_LAUNCH(k_ref_terms<T>, blocks_for(last - first, 256), 256, 0, s, make_gridk<T>(*g), R,
               (T)rho, gR, nR, first, last);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int ngf_terms_impl(const ngf_grid_t* g, const T* W, const T* gR, const T* nR, double tau,
                   double rho, T* terms, T* q, cudaStream_t s) {
    const T taut = (T)tau;
    const double hbar = g->spacing[0] * g->spacing[1] * g->spacing[2];
    NGF_LAUNCH(k_ngf_terms<T>, blocks_for(grid_n(*g), 256), 256, 0, s, make_gridk<T>(*g), W, gR,
               nR, taut * taut, (T)(tau * rho), (T)(-hbar), terms, q);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int laplacian_impl(const ngf_grid_t* g, const T* u, T* out, int ncomp, cudaStream_t s) {
    NGF_LAUNCH(k_laplacian<T>, blocks_for(grid_n(*g) * ncomp, 256), 256, 0, s, make_gridk<T>(*g), u,
               out, ncomp);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int laplacian_t_impl(const ngf_grid_t* g, const T* w, T* out, int ncomp, T scale, int use_scale,
                     const T* add, T add_scale, cudaStream_t s) {
    NGF_LAUNCH(k_laplacian_t<T>, blocks_for(grid_n(*g) * ncomp, 256), 256, 0, s, make_gridk<T>(*g),
               w, out, ncomp, scale, use_scale, add, add_scale, (T*)nullptr);
    NGF_CHECK_LAUNCH();
    return 0;
}

// S (to S_dev) and grad = [add +] f(alpha) * vol * L^T L u; workspace: 2 * 3M of T + 3 doubles
template <typename T>
int curvature_impl(const ngf_grid_t* g, const T* y, double* S_dev, T* grad, const T* add,
                   double alpha, T* ws, double* ws_d, cudaStream_t s) {
    const int64_t m = grid_n(*g);
    GridK<T> gk = make_gridk<T>(*g);
    T* u = ws;
    T* L = ws + 3 * m;
    NGF_LAUNCH(k_displacement<T>, blocks_for(3 * m, 256), 256, 0, s, gk, y, u);
    int rc = laplacian_impl<T>(g, u, L, 3, s);
    if (rc) return rc;
    const double vol = g->spacing[0] * g->spacing[1] * g->spacing[2];
    if (S_dev) {
        // per component pairwise sum of L*L, then the f32/f64 running total (curvature.py:66-71)
        NGF_LAUNCH(k_square<T>, blocks_for(3 * m, 256), 256, 0, s, L, u, 3 * m);  // u <- L*L
        for (int c = 0; c < 3; ++c) {
            rc = pairwise_sum_impl<T>(u + c * m, m, ws_d + c, 0, 0.0, s);
            if (rc) return rc;
        }
        NGF_LAUNCH(k_curv_total<T>, 1, 1, 0, s, ws_d, vol / 2, S_dev);
    }
    if (grad) {
        // out = vol * L^T (L u) ; objective adds grad_D + f(alpha) * that (objective.py:50)
        rc = laplacian_t_impl<T>(g, L, grad, 3, (T)vol, 1, add, (T)alpha, s);
        if (rc) return rc;
    }
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int downsample_impl(const ngf_grid_t* g, const T* in, T* out, cudaStream_t s) {
    const int nx = (int)g->dims[0], ny = (int)g->dims[1], nz = (int)g->dims[2];
    const int64_t m = (int64_t)(nx > 1 ? (nx + 1) / 2 : 1) * (ny > 1 ? (ny + 1) / 2 : 1) *
                      (nz > 1 ? (nz + 1) / 2 : 1);
    NGF_LAUNCH(k_downsample<T>, blocks_for(m, 256), 256, 0, s, nx, ny, nz, in, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int prolong_impl(const ngf_plan_t* p, const T* yc, T* yf, cudaStream_t s) {
    if (int rc = plan_upload(const_cast<ngf_plan_t*>(p))) return rc;
    const int64_t n = grid_n(p->img_grid);
    NGF_LAUNCH(k_prolong<T>, blocks_for(n, 256), 256, 0, s, p->axes[0], p->axes[1], p->axes[2],
               make_gridk<T>(p->def_grid), make_gridk<T>(p->img_grid), yc, yf);
    NGF_CHECK_LAUNCH();
    return 0;
}

// ------------------------------------------------------------------ deformation probes
// Trilinear value of the 3-component field at world points, clamp-to-edge, in f64
// (evaluation.py:39-64: t = (p - o) / h, i0 = clip(floor t, 0, max(n - 2, 0)),
// f = clip(t - i0, 0, 1) (0 on a one-node axis), terms accumulated dz, dy, dx with
// w = (wx * wy) * wz).
template <typename T>
__global__ void k_sample_field(GridK<T> g, const T* __restrict__ y, const double* __restrict__ pts, int64_t n,
                               double* __restrict__ out) {
    const int64_t m = (int64_t)g.nx * g.ny * g.nz;
    const int dims[3] = {g.nx, g.ny, g.nz};
    const double org[3] = {g.dox, g.doy, g.doz}, sp[3] = {g.dhx, g.dhy, g.dhz};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        int i0[3];
        double f[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double t = (pts[3 * p + a] - org[a]) / sp[a];
            const int hi = dims[a] > 2 ? dims[a] - 2 : 0;
            const double fl = floor(t);
            const int i = fl < 0.0 ? 0 : (fl > (double)hi ? hi : (int)fl);
            i0[a] = i;
            const double fr = t - (double)i;
            f[a] = dims[a] > 1 ? fmin(fmax(fr, 0.0), 1.0) : 0.0;
        }
        double acc[3] = {0.0, 0.0, 0.0};
        for (int dz = 0; dz < 2; ++dz) {
            const double wz = dz ? f[2] : 1.0 - f[2];
            const int iz = min(i0[2] + dz, g.nz - 1);
            for (int dy = 0; dy < 2; ++dy) {
                const double wy = dy ? f[1] : 1.0 - f[1];
                const int iy = min(i0[1] + dy, g.ny - 1);
                for (int dx = 0; dx < 2; ++dx) {
                    const double wx = dx ? f[0] : 1.0 - f[0];
                    const int ix = min(i0[0] + dx, g.nx - 1);
                    const double w = (wx * wy) * wz;
                    const int64_t idx = ((int64_t)iz * g.ny + iy) * g.nx + ix;
#pragma unroll
                    for (int c = 0; c < 3; ++c) acc[c] = acc[c] + w * (double)y[c * m + idx];
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) out[3 * p + c] = acc[c];
    }
}

template <typename T>
int sample_field_impl(const ngf_grid_t* g, const T* y, const double* pts, int64_t n, double* out, cudaStream_t s) {
    if (n == 0) return 0;
    NGF_LAUNCH(k_sample_field<T>, blocks_for(n, 128), 128, 0, s, make_gridk<T>(*g), y, pts, n, out);
    NGF_CHECK_LAUNCH();
    return 0;
}

// explicit instantiations
#define NGF_INST(T)                                                                              \
    template int apply_P_impl<T>(const ngf_plan_t*, const T*, T*, cudaStream_t);                 \
    template int apply_Pt_impl<T>(const ngf_plan_t*, const T*, T*, cudaStream_t);                \
    template int apply_Pt_variant_impl<T>(const ngf_plan_t*, int, const T*, T*, cudaStream_t);   \
    template int warp_impl<T>(const ngf_grid_t*, const T*, const T*, int64_t, T*, uint8_t*,      \
                              cudaStream_t);                                                     \
    template int warp_jt_impl<T>(const ngf_grid_t*, const T*, const T*, const T*, int64_t, T*,  \
                                 cudaStream_t);                                                  \
    template int gradient_impl<T>(const ngf_grid_t*, const T*, T*, cudaStream_t);               \
    template int gradient_t_impl<T>(const ngf_grid_t*, const T*, T*, cudaStream_t);             \
    template int ref_terms_impl<T>(const ngf_grid_t*, const T*, double, T*, T*, cudaStream_t, int64_t, int64_t); \
    template int ngf_terms_impl<T>(const ngf_grid_t*, const T*, const T*, const T*, double,     \
                                   double, T*, T*, cudaStream_t);                               \
    template int pairwise_sum_impl<T>(const T*, int64_t, double*, int, double, cudaStream_t);    \
    template int laplacian_impl<T>(const ngf_grid_t*, const T*, T*, int, cudaStream_t);         \
    template int laplacian_t_impl<T>(const ngf_grid_t*, const T*, T*, int, T, int, const T*, T,  \
                                     cudaStream_t);                                             \
    template int curvature_impl<T>(const ngf_grid_t*, const T*, double*, T*, const T*, double,  \
                                   T*, double*, cudaStream_t);                                  \
    template int downsample_impl<T>(const ngf_grid_t*, const T*, T*, cudaStream_t);             \
    template int prolong_impl<T>(const ngf_plan_t*, const T*, T*, cudaStream_t);                 \
    template int sample_field_impl<T>(const ngf_grid_t*, const T*, const double*, int64_t, double*, \
                                      cudaStream_t);

NGF_INST(float)
NGF_INST(double)

}  // namespace ngf
