// Fused NGF objective/gradient evaluation for sm_100a (the performance path).
//
// One CTA owns a kTX x kTY column of image voxels plus a one-voxel ring
// (E1 = (kTX+2) x (kTY+2) positions, kSlots per thread) and marches a chunk of
// z-planes.  Step p of the march
//   (A) interpolates yhat = P y on the fly for plane p (bit-exact with transfer.py:
//       117-148, so the inside/floor decisions of warp.py:32-53 match the
//       reference), gathers the 8 template corners of every slot at once and forms
//       W (warp.py:64-90) and the interpolant derivative / h (warp.py:93-127);
//   (B) forms grad W (warp.py:130-143), the NGF ratio, the distance term and
//       q = dD/d(grad W) (ngf.py:70-112) on the tile interior for plane p-1, with
//       the packed reference terms prefetched one step ahead;
//   (C) applies G^T (warp.py:159-184) and the warp Jacobian transpose for plane p-2
//       and accumulates P^T along z in registers (transfer.py:151-192 with the
//       axes reordered z-first); when a deformation plane is complete, the CTA
//       reduces it in x then y in a fixed order and writes its window partial.
// yhat, W, grad W, q, s and ghat never leave the SM.  G^T and P^T are linear, so
// ring voxels carry only this tile's contributions; k_reduce adds the tiles that
// share a deformation node in a fixed order (deterministic, no atomics).

#include <vector>

#include "common.cuh"
#include "eval_fused.cuh"
#include "fused_impl.cuh"

namespace ngf {

template <typename T>
__device__ __forceinline__ void fd_coef(int i, int n, T ih, T& cm, T& c0, T& cp) {
    // derivative at index i as cm*v[i-1] + c0*v[i] + cp*v[i+1] (warp.py:130-143)
    cm = (T)0;
    c0 = (T)0;
    cp = (T)0;
    if (n < 2 || i < 0 || i >= n) return;
    if (i == 0) {
        c0 = -ih;
        cp = ih;
    } else if (i == n - 1) {
        cm = -ih;
        c0 = ih;
    } else {
        cm = (T)-0.5 * ih;
        cp = (T)0.5 * ih;
    }
}

// transpose coefficients at index i: multiply q[i-1], q[i], q[i+1]
template <typename T>
__device__ __forceinline__ void fdt_coef(int i, int n, T ih, T& gm, T& g0, T& gp) {
    T a, b, c;
    fd_coef<T>(i - 1, n, ih, a, b, c);
    gm = c;
    fd_coef<T>(i, n, ih, a, b, c);
    g0 = b;
    fd_coef<T>(i + 1, n, ih, a, b, c);
    gp = a;
}

template <typename T>
struct Smem {
    T* colG;    // [kE1X][3]  G coefficients (cm, c0, cp)
    T* colGt;   // [kE1X][3]  G^T coefficients
    T* rowG;    // [kE1Y][3]
    T* rowGt;   // [kE1Y][3]
    T* colPw;   // [kE1X]     P weight wx (dtype)
    T* rowPw;   // [kE1Y]
    T* Wsm;     // [3][kE1]   W ring (planes p-2, p-1, p)
    T* qx;      // [3][kE2]   q_x ring, zero-padded
    T* qy;      // [3][kE2]
    T* buf;     // [3][kE1]   completed deformation plane (z-reduced ghat)
    T* Xr;      // [3][kE1Y][wx] x-reduced
    T* xw;      // [2*kE1X]   CSR weights, window column d <- E1 columns
    T* yw;      // [2*kE1Y]
    int* colP0;  // [kE1X] P: def x0, x1
    int* colP1;
    int* rowP0;
    int* rowP1;
    int* xoff;  // [wx+1]
    int* xcol;  // [2*kE1X]
    int* yoff;  // [wy+1]
    int* yrow;  // [2*kE1Y]
    double* red;  // [kThreads/32]
};

template <typename T>
__device__ __forceinline__ T* carve(unsigned char*& p, size_t count) {
    size_t bytes = (count * sizeof(T) + 15) & ~size_t(15);
    T* q = reinterpret_cast<T*>(p);
    p += bytes;
    return q;
}

template <typename T>
__host__ __device__ inline size_t fused_smem_bytes(int wx, int wy, int wz) {
    auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
    (void)wz;
    size_t s = 0;
    s += al(kE1X * 3 * sizeof(T)) * 2 + al(kE1Y * 3 * sizeof(T)) * 2;
    s += al(kE1X * sizeof(T)) + al(kE1Y * sizeof(T));
    s += al(3 * kE1 * sizeof(T));
    s += al(3 * kE2 * sizeof(T)) * 2;
    s += al(3 * kE1 * sizeof(T));
    s += al((size_t)3 * kE1Y * wx * sizeof(T));
    s += al(2 * kE1X * sizeof(T)) + al(2 * kE1Y * sizeof(T));
    s += al(kE1X * 4) * 2 + al(kE1Y * 4) * 2;
    s += al((wx + 1) * 4) + al(2 * kE1X * 4) + al((wy + 1) * 4) + al(2 * kE1Y * 4);
    s += al((kThreads / 32) * 8);
    return s;
}

template <typename T>
__device__ __forceinline__ Smem<T> carve_smem(unsigned char* base, int wx, int wy) {
    Smem<T> s;
    unsigned char* p = base;
    s.colG = carve<T>(p, kE1X * 3);
    s.colGt = carve<T>(p, kE1X * 3);
    s.rowG = carve<T>(p, kE1Y * 3);
    s.rowGt = carve<T>(p, kE1Y * 3);
    s.colPw = carve<T>(p, kE1X);
    s.rowPw = carve<T>(p, kE1Y);
    s.Wsm = carve<T>(p, 3 * kE1);
    s.qx = carve<T>(p, 3 * kE2);
    s.qy = carve<T>(p, 3 * kE2);
    s.buf = carve<T>(p, 3 * kE1);
    s.Xr = carve<T>(p, (size_t)3 * kE1Y * wx);
    s.xw = carve<T>(p, 2 * kE1X);
    s.yw = carve<T>(p, 2 * kE1Y);
    s.colP0 = carve<int>(p, kE1X);
    s.colP1 = carve<int>(p, kE1X);
    s.rowP0 = carve<int>(p, kE1Y);
    s.rowP1 = carve<int>(p, kE1Y);
    s.xoff = carve<int>(p, wx + 1);
    s.xcol = carve<int>(p, 2 * kE1X);
    s.yoff = carve<int>(p, wy + 1);
    s.yrow = carve<int>(p, 2 * kE1Y);
    s.red = carve<double>(p, kThreads / 32);
    return s;
}

// Per-thread march state.  Slot s owns E1 position P = tid + s * kThreads for all planes.
template <typename T>
struct March {
    int P[kSlots];     // flat E1 index (-1: no position)
    int P2[kSlots];    // index in the zero-padded q layout
    int ij[kSlots];    // j * nx + i of the image column (RT / volume offset in a plane)
    int exy[kSlots];   // ex | ey << 8
    unsigned flags;    // bit s: inside the image in x/y; bit 8+s: tile interior
    T ylo[kSlots][3], yhi[kSlots][3];   // P_xy y on the current def-plane pair
    T dT[kSlots][3][3];                 // interpolant derivative / h, plane ring
    T qz[kSlots][3];                    // q_z, plane ring
    T A0[kSlots][3], A1[kSlots][3];     // z-accumulated ghat for def planes zd, zd+1
    V4T<T> rt[kSlots];                  // prefetched reference terms (next B plane)
    int z0, z1, jfirst, jlast, wxlo, wylo, wzlo, cur_zd, cta;
    double dacc;
};

template <typename T>
__device__ __forceinline__ bool slot_vol(const March<T>& m, int s) { return (m.flags >> s) & 1u; }
template <typename T>
__device__ __forceinline__ bool slot_e0(const March<T>& m, int s) { return (m.flags >> (8 + s)) & 1u; }

template <typename T>
__device__ __forceinline__ void load_yplane(const FusedArgs<T>& a, const Smem<T>& sm, int exy, int zd,
                                            T (&out)[3]) {
    // P_xy y on def plane zd at the slot's image (i, j): x then y (transfer.py:136-142)
    const int ex = exy & 0xff, ey = exy >> 8;
    const int x0 = sm.colP0[ex], x1 = sm.colP1[ex];
    const int y0 = sm.rowP0[ey], y1 = sm.rowP1[ey];
    const T wx = sm.colPw[ex], wy = sm.rowPw[ey];
    const int64_t mm = (int64_t)a.ndx * a.ndy * a.ndz;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* yc = a.y + k * mm + (int64_t)zd * a.ndx * a.ndy;
        const T* r0 = yc + (int64_t)y0 * a.ndx;
        const T* r1 = yc + (int64_t)y1 * a.ndx;
        const T X0 = lerp_exact(__ldg(r0 + x0), __ldg(r0 + x1), wx);
        const T X1 = lerp_exact(__ldg(r1 + x0), __ldg(r1 + x1), wx);
        out[k] = lerp_exact(X0, X1, wy);
    }
}

// Reduce a completed deformation plane (z-accumulated ghat in `acc`) in x then y over
// the tile's window and write it to the CTA's partial slot zs.
template <typename T>
__device__ __forceinline__ void flush_plane(const FusedArgs<T>& a, const Smem<T>& sm, March<T>& m,
                                            T (&acc)[kSlots][3], int zs) {
    const int wx = a.fp.wx, wy = a.fp.wy;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
        if (m.P[s] < 0) continue;
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.buf[c * kE1 + m.P[s]] = acc[s][c];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kE1Y * wx; t += kThreads) {
        const int row = t / wx;
        const int d = t - row * wx;
        const int k0 = sm.xoff[d], k1 = sm.xoff[d + 1];
        T r0 = (T)0, r1 = (T)0, r2 = (T)0;
        const T* b = sm.buf + row * kE1X;
        for (int k = k0; k < k1; ++k) {
            const int e = sm.xcol[k];
            const T w = sm.xw[k];
            r0 = fmaf_t(b[e], w, r0);
            r1 = fmaf_t(b[kE1 + e], w, r1);
            r2 = fmaf_t(b[2 * kE1 + e], w, r2);
        }
        sm.Xr[(0 * kE1Y + row) * wx + d] = r0;
        sm.Xr[(1 * kE1Y + row) * wx + d] = r1;
        sm.Xr[(2 * kE1Y + row) * wx + d] = r2;
    }
    __syncthreads();
    const size_t win = (size_t)a.fp.wz * wy * wx;
    T* out = a.partial + (size_t)m.cta * 3 * win + (size_t)zs * wy * wx;
    for (int t = threadIdx.x; t < wy * wx; t += kThreads) {
        const int dr = t / wx;
        const int d = t - dr * wx;
        const int k0 = sm.yoff[dr], k1 = sm.yoff[dr + 1];
        T r0 = (T)0, r1 = (T)0, r2 = (T)0;
        for (int k = k0; k < k1; ++k) {
            const int row = sm.yrow[k];
            const T w = sm.yw[k];
            r0 = fmaf_t(sm.Xr[(0 * kE1Y + row) * wx + d], w, r0);
            r1 = fmaf_t(sm.Xr[(1 * kE1Y + row) * wx + d], w, r1);
            r2 = fmaf_t(sm.Xr[(2 * kE1Y + row) * wx + d], w, r2);
        }
        out[t] = r0;
        out[win + t] = r1;
        out[2 * win + t] = r2;
    }
}

template <int R, typename T>
__device__ __forceinline__ void fused_step(const FusedArgs<T>& a, const Smem<T>& sm, March<T>& m,
                                           int p) {
    constexpr int RB = (R + 2) % 3;  // plane p-1
    constexpr int RC = (R + 1) % 3;  // plane p-2

    // ---------------------------------------------------------------- (A) plane p
    if (p >= 0 && p < a.nz && p <= m.z1) {
        const int zd = a.i0z[p];
        if (zd != m.cur_zd) {
            const int zd1 = min(zd + 1, a.ndz - 1);
            const bool shift = (zd == m.cur_zd + 1);
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
                if (!slot_vol(m, s)) continue;
                if (shift) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) m.ylo[s][k] = m.yhi[s][k];
                } else {
                    load_yplane(a, sm, m.exy[s], zd, m.ylo[s]);
                }
                load_yplane(a, sm, m.exy[s], zd1, m.yhi[s]);
            }
            m.cur_zd = zd;
        }
        const T wz = a.w1z[p];
        // coordinates and corner addresses of all slots first, so the 8 * kSlots
        // gathers are in flight together
        const T* base[kSlots];
        T fx[kSlots], fy[kSlots], fz[kSlots];
        bool in[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
            T yh0 = lerp_exact(m.ylo[s][0], m.yhi[s][0], wz);
            T yh1 = lerp_exact(m.ylo[s][1], m.yhi[s][1], wz);
            T yh2 = lerp_exact(m.ylo[s][2], m.yhi[s][2], wz);
            bool inside = slot_vol(m, s);
            int ix, iy, iz;
            axis_cell(tcoord(yh0, a.ox, a.hx, a.ihx, a.pow2x), a.nx, inside, ix, fx[s]);
            axis_cell(tcoord(yh1, a.oy, a.hy, a.ihy, a.pow2y), a.ny, inside, iy, fy[s]);
            axis_cell(tcoord(yh2, a.oz, a.hz, a.ihz, a.pow2z), a.nz, inside, iz, fz[s]);
            in[s] = inside;
            base[s] = a.Tv + ((int64_t)iz * a.ny + iy) * a.nx + ix;
        }
        const int64_t sx = a.nx > 1 ? 1 : 0;
        const int64_t sy = a.ny > 1 ? a.nx : 0;
        const int64_t sz = a.nz > 1 ? (int64_t)a.nx * a.ny : 0;
        T cv[kSlots][8];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
            const T* b = base[s];
            cv[s][0] = __ldg(b);
            cv[s][1] = __ldg(b + sx);
            cv[s][2] = __ldg(b + sy);
            cv[s][3] = __ldg(b + sy + sx);
            cv[s][4] = __ldg(b + sz);
            cv[s][5] = __ldg(b + sz + sx);
            cv[s][6] = __ldg(b + sz + sy);
            cv[s][7] = __ldg(b + sz + sy + sx);
        }
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
            T W, d0, d1, d2;
            trilinear(a, cv[s], fx[s], fy[s], fz[s], W, d0, d1, d2);
            if (!in[s]) W = d0 = d1 = d2 = (T)0;
            m.dT[s][R][0] = d0;
            m.dT[s][R][1] = d1;
            m.dT[s][R][2] = d2;
            if (m.P[s] >= 0) sm.Wsm[R * kE1 + m.P[s]] = W;
        }
    } else {
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
            m.dT[s][R][0] = m.dT[s][R][1] = m.dT[s][R][2] = (T)0;
            if (m.P[s] >= 0) sm.Wsm[R * kE1 + m.P[s]] = (T)0;
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (B) q on plane k = p-1
    {
        const int k = p - 1;
        const bool kv = (k >= m.z0) && (k < m.z1);
        T cmz, c0z, cpz;
        fd_coef<T>(k, a.nz, a.ihz, cmz, c0z, cpz);
        const T* Wk = sm.Wsm + RB * kE1;
        const T* Wm = sm.Wsm + RC * kE1;
        const T* Wp = sm.Wsm + R * kE1;
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
            T qxv = (T)0, qyv = (T)0, qzv = (T)0;
            if (kv && slot_e0(m, s)) {
                const int P = m.P[s];
                const int ex = m.exy[s] & 0xff, ey = m.exy[s] >> 8;
                const T* cg = sm.colG + 3 * ex;
                const T* rg = sm.rowG + 3 * ey;
                const T gx = fmaf_t(cg[0], Wk[P - 1], fmaf_t(cg[1], Wk[P], cg[2] * Wk[P + 1]));
                const T gy = fmaf_t(rg[0], Wk[P - kE1X], fmaf_t(rg[1], Wk[P], rg[2] * Wk[P + kE1X]));
                const T gz = fmaf_t(cmz, Wm[P], fmaf_t(c0z, Wk[P], cpz * Wp[P]));
                ngf_q(a, gx, gy, gz, m.rt[s], qxv, qyv, qzv, m.dacc);
            }
            if (m.P[s] >= 0) {
                sm.qx[RB * kE2 + m.P2[s]] = qxv;
                sm.qy[RB * kE2 + m.P2[s]] = qyv;
            }
            m.qz[s][RB] = qzv;
        }
        // prefetch the reference terms of plane p for the next step's (B)
        if (p >= m.z0 && p < m.z1) {
            const V4T<T>* rp = a.RT + (int64_t)p * a.nx * a.ny;
#pragma unroll
            for (int s = 0; s < kSlots; ++s)
                if (slot_e0(m, s)) m.rt[s] = ld_rt(rp + m.ij[s]);
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (C) s, ghat, z-P^T on j = p-2
    const int j = p - 2;
    if (j < m.jfirst || j > m.jlast) return;  // uniform
    T gtm, gt0, gtp;
    fdt_coef<T>(j, a.nz, a.ihz, gtm, gt0, gtp);
    const T* qxj = sm.qx + RC * kE2;
    const T* qyj = sm.qy + RC * kE2;
    const int zdj = a.i0z[j];
    const T w1 = a.w1z[j];
    const T w0 = (T)1 - w1;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
        if (!slot_vol(m, s)) continue;
        const int P2 = m.P2[s];
        const int ex = m.exy[s] & 0xff, ey = m.exy[s] >> 8;
        const T* ct = sm.colGt + 3 * ex;
        const T* rt = sm.rowGt + 3 * ey;
        T sv = fmaf_t(ct[0], qxj[P2 - 1], fmaf_t(ct[1], qxj[P2], ct[2] * qxj[P2 + 1]));
        sv = fmaf_t(rt[0], qyj[P2 - kE2X], fmaf_t(rt[1], qyj[P2], fmaf_t(rt[2], qyj[P2 + kE2X], sv)));
        sv = fmaf_t(gtm, m.qz[s][R], fmaf_t(gt0, m.qz[s][RC], fmaf_t(gtp, m.qz[s][RB], sv)));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T g = sv * m.dT[s][RC][c];
            m.A0[s][c] = fmaf_t(w0, g, m.A0[s][c]);
            m.A1[s][c] = fmaf_t(w1, g, m.A1[s][c]);
        }
    }
    // def plane zdj is complete when the next image plane maps to a later pair.  The map
    // can advance by 2 (w1 rounds to just below 1 when the grids nearly coincide), in
    // which case zdj + 1 is complete as well.
    const bool last = (j == m.jlast);
    const int step = last ? 2 : a.i0z[j + 1] - zdj;
    if (step >= 1) {
        flush_plane(a, sm, m, m.A0, zdj - m.wzlo);
        if (step >= 2) {
            if (zdj + 1 <= a.ndz - 1) {
                __syncthreads();
                flush_plane(a, sm, m, m.A1, zdj + 1 - m.wzlo);
            }
#pragma unroll
            for (int s = 0; s < kSlots; ++s)
#pragma unroll
                for (int c = 0; c < 3; ++c) m.A0[s][c] = m.A1[s][c] = (T)0;
        } else {
#pragma unroll
            for (int s = 0; s < kSlots; ++s)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    m.A0[s][c] = m.A1[s][c];
                    m.A1[s][c] = (T)0;
                }
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) k_eval_fused(const __grid_constant__ FusedArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const FusedPlan& fp = a.fp;
    const Smem<T> sm = carve_smem<T>(smem_raw, fp.wx, fp.wy);
    const int tid = threadIdx.x;
    March<T> m;
    m.cta = blockIdx.x;
    const int tx = m.cta % fp.ntx;
    const int ty = (m.cta / fp.ntx) % fp.nty;
    const int tz = m.cta / (fp.ntx * fp.nty);
    const int x0 = tx * kTX, y0 = ty * kTY;
    m.z0 = tz * fp.cz;
    m.z1 = min(m.z0 + fp.cz, a.nz);
    m.jfirst = max(m.z0 - 1, 0);
    m.jlast = min(m.z1, a.nz - 1);
    m.wxlo = fp.win_x[tx];
    m.wylo = fp.win_y[ty];
    m.wzlo = fp.win_z[tz];
    m.cur_zd = -1000;
    m.dacc = 0.0;

    // ---- per-CTA tables
    for (int e = tid; e < kE1X; e += kThreads) {
        const int i = x0 - 1 + e;
        T cm, c0, cp;
        fd_coef<T>(i, a.nx, a.ihx, cm, c0, cp);
        sm.colG[3 * e] = cm;
        sm.colG[3 * e + 1] = c0;
        sm.colG[3 * e + 2] = cp;
        fdt_coef<T>(i, a.nx, a.ihx, cm, c0, cp);
        sm.colGt[3 * e] = cm;
        sm.colGt[3 * e + 1] = c0;
        sm.colGt[3 * e + 2] = cp;
        const bool in = i >= 0 && i < a.nx;
        const int i0 = in ? a.i0x[i] : 0;
        sm.colP0[e] = i0;
        sm.colP1[e] = min(i0 + 1, a.ndx - 1);
        sm.colPw[e] = in ? a.w1x[i] : (T)0;
    }
    for (int e = tid; e < kE1Y; e += kThreads) {
        const int jj = y0 - 1 + e;
        T cm, c0, cp;
        fd_coef<T>(jj, a.ny, a.ihy, cm, c0, cp);
        sm.rowG[3 * e] = cm;
        sm.rowG[3 * e + 1] = c0;
        sm.rowG[3 * e + 2] = cp;
        fdt_coef<T>(jj, a.ny, a.ihy, cm, c0, cp);
        sm.rowGt[3 * e] = cm;
        sm.rowGt[3 * e + 1] = c0;
        sm.rowGt[3 * e + 2] = cp;
        const bool in = jj >= 0 && jj < a.ny;
        const int i0 = in ? a.i0y[jj] : 0;
        sm.rowP0[e] = i0;
        sm.rowP1[e] = min(i0 + 1, a.ndy - 1);
        sm.rowPw[e] = in ? a.w1y[jj] : (T)0;
    }
    for (int t = tid; t < 3 * kE2; t += kThreads) {
        sm.qx[t] = (T)0;
        sm.qy[t] = (T)0;
    }
    if (tid == 0 || tid == 32) {
        // CSR of the transposed 1-D interpolation over the tile window, ascending
        // E1 index per window entry (the reference's gather order, transfer.py:89-96)
        const bool isx = tid == 0;
        const int ne = isx ? kE1X : kE1Y, w = isx ? fp.wx : fp.wy, org = isx ? x0 : y0;
        const int n = isx ? a.nx : a.ny, nd = isx ? a.ndx : a.ndy, lo = isx ? m.wxlo : m.wylo;
        const int32_t* i0a = isx ? a.i0x : a.i0y;
        const T* w1a = isx ? a.w1x : a.w1y;
        int* off = isx ? sm.xoff : sm.yoff;
        int* idx = isx ? sm.xcol : sm.yrow;
        T* wt = isx ? sm.xw : sm.yw;
        int cnt = 0;
        for (int d = 0; d < w; ++d) {
            off[d] = cnt;
            for (int e = 0; e < ne; ++e) {
                const int i = org - 1 + e;
                if (i < 0 || i >= n) continue;
                const int dl = i0a[i] - lo;
                const T w1 = w1a[i];
                if (dl == d) {
                    idx[cnt] = e;
                    wt[cnt++] = (T)1 - w1;
                } else if (dl == d - 1 && nd > 1) {
                    idx[cnt] = e;
                    wt[cnt++] = w1;
                }
            }
        }
        off[w] = cnt;
    }

    // ---- slot positions (fixed for all planes)
    m.flags = 0u;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) {
        const int P = tid + s * kThreads;
        const bool ok = P < kE1;
        const int ex = ok ? P % kE1X : 0, ey = ok ? P / kE1X : 0;
        const int i = x0 - 1 + ex, jj = y0 - 1 + ey;
        const bool vol = ok && i >= 0 && i < a.nx && jj >= 0 && jj < a.ny;
        const bool e0 = vol && ex >= 1 && ex <= kTX && ey >= 1 && ey <= kTY;
        m.P[s] = ok ? P : -1;
        m.P2[s] = (ey + 1) * kE2X + ex + 1;
        m.ij[s] = vol ? jj * a.nx + i : 0;
        m.exy[s] = ex | (ey << 8);
        m.flags |= (vol ? 1u : 0u) << s;
        m.flags |= (e0 ? 1u : 0u) << (8 + s);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            m.qz[s][r] = (T)0;
            m.dT[s][r][0] = m.dT[s][r][1] = m.dT[s][r][2] = (T)0;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            m.ylo[s][c] = m.yhi[s][c] = (T)0;
            m.A0[s][c] = m.A1[s][c] = (T)0;
        }
        m.rt[s] = V4T<T>{};
    }
    __syncthreads();
    // reference terms of the first interior plane
    if (m.z0 < m.z1) {
        const V4T<T>* rp = a.RT + (int64_t)m.z0 * a.nx * a.ny;
#pragma unroll
        for (int s = 0; s < kSlots; ++s)
            if (slot_e0(m, s)) m.rt[s] = ld_rt(rp + m.ij[s]);
    }

    // planes p = z0-1 .. z1+2: (A) on p, (B) on p-1, (C) on p-2
    const int pstart = m.z0 - 1;
    const int nsteps = (m.z1 + 2) - pstart + 1;
    for (int b = 0; b < nsteps; b += 3) {
        fused_step<0>(a, sm, m, pstart + b);
        if (b + 1 < nsteps) fused_step<1>(a, sm, m, pstart + b + 1);
        if (b + 2 < nsteps) fused_step<2>(a, sm, m, pstart + b + 2);
    }

    // ---- the CTA's D partial
    double v = m.dacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) sm.red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
        double sacc = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) sacc += sm.red[w];
        a.dpart[m.cta] = sacc;
    }
}

// ------------------------------------------------------------------ reduce + curvature

// Lu (3, M) of the displacement and per-block partial sums of (Lu)^2
template <typename T>
__global__ void k_curv_L(GridK<T> g, const T* __restrict__ y, T* __restrict__ L,
                         double* __restrict__ spart, int* __restrict__ flag) {
    const int64_t m = g.n();
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const T ihx2 = (T)1 / (g.hx * g.hx), ihy2 = (T)1 / (g.hy * g.hy), ihz2 = (T)1 / (g.hz * g.hz);
    double acc = 0.0;
    bool bad = false;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * m;
         t += (int64_t)gridDim.x * blockDim.x) {
        bad |= !isfinite(y[t]);
        const int comp = (int)(t / m);
        const int64_t idx = t % m;
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        const T* yc = y + comp * m;
        auto u = [&](int ii, int jj, int kk) -> T {
            const T idv = comp == 0 ? (T)(g.dox + g.dhx * (double)ii)
                                    : (comp == 1 ? (T)(g.doy + g.dhy * (double)jj)
                                                 : (T)(g.doz + g.dhz * (double)kk));
            return yc[((int64_t)kk * g.ny + jj) * g.nx + ii] - idv;
        };
        const T u0 = u(i, j, k);
        T lap = (T)0;
        if (g.nx >= 3 && i > 0 && i < g.nx - 1) lap += (u(i + 1, j, k) - (T)2 * u0 + u(i - 1, j, k)) * ihx2;
        if (g.ny >= 3 && j > 0 && j < g.ny - 1) lap += (u(i, j + 1, k) - (T)2 * u0 + u(i, j - 1, k)) * ihy2;
        if (g.nz >= 3 && k > 0 && k < g.nz - 1) lap += (u(i, j, k + 1) - (T)2 * u0 + u(i, j, k - 1)) * ihz2;
        L[t] = lap;
        acc += (double)lap * (double)lap;
        (void)sy;
    }
    __shared__ double red[32];
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        spart[blockIdx.x] = s;
    }
}

template <typename T>
__device__ __forceinline__ T d2t(const T* w, int64_t idx, int i, int n, int64_t stride, T ih2) {
    if (n < 3) return (T)0;
    T o = (T)0;
    if (i <= n - 3) o += w[idx + stride];
    if (i >= 1 && i <= n - 2) o -= (T)2 * w[idx];
    if (i >= 2) o += w[idx - stride];
    return o * ih2;
}

template <typename T>
__global__ void k_reduce(GridK<T> g, const FusedPlan fp, const T* __restrict__ partial,
                         const T* __restrict__ L, T vol, T alpha, T* __restrict__ grad) {
    const int64_t m = g.n();
    const int64_t sz = (int64_t)g.nx * g.ny;
    const int win = fp.wz * fp.wy * fp.wx;
    const T ihx2 = (T)1 / (g.hx * g.hx), ihy2 = (T)1 / (g.hy * g.hy), ihz2 = (T)1 / (g.hz * g.hz);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 3 * m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int comp = (int)(t / m);
        const int64_t idx = t % m;
        const int i = (int)(idx % g.nx);
        const int j = (int)((idx / g.nx) % g.ny);
        const int k = (int)(idx / sz);
        // grad D: fixed-order sum of the covering tiles' partials
        T gd = (T)0;
        const int32_t* cz = fp.cov_z + (int64_t)k * kCover * 2;
        const int32_t* cy = fp.cov_y + (int64_t)j * kCover * 2;
        const int32_t* cx = fp.cov_x + (int64_t)i * kCover * 2;
        for (int az = 0; az < kCover && cz[2 * az] >= 0; ++az) {
            for (int ay = 0; ay < kCover && cy[2 * ay] >= 0; ++ay) {
                for (int ax = 0; ax < kCover && cx[2 * ax] >= 0; ++ax) {
                    const int cta = (cz[2 * az] * fp.nty + cy[2 * ay]) * fp.ntx + cx[2 * ax];
                    const int off = (cz[2 * az + 1] * fp.wy + cy[2 * ay + 1]) * fp.wx + cx[2 * ax + 1];
                    gd += __ldg(partial + ((size_t)cta * 3 + comp) * win + off);
                }
            }
        }
        // grad S = vol * L^T L u (curvature.py:74-81)
        const T* Lc = L + comp * m;
        T lt = d2t(Lc, idx, i, g.nx, 1, ihx2) + d2t(Lc, idx, j, g.ny, (int64_t)g.nx, ihy2) +
               d2t(Lc, idx, k, g.nz, sz, ihz2);
        grad[t] = gd + alpha * (vol * lt);
    }
}

template <typename T>
__global__ void k_finalize(const double* __restrict__ dpart, int nd, const double* __restrict__ spart,
                           int ns, double half_hbar, double half_vol, double alpha, int* flag,
                           double* __restrict__ out) {
    // fixed-order sums; D and S rounded like the reference's dtype products
    __shared__ double red[2][32];
    double a = 0.0, b = 0.0;
    for (int t = threadIdx.x; t < nd; t += blockDim.x) a += dpart[t];
    for (int t = threadIdx.x; t < ns; t += blockDim.x) b += spart[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = a;
        red[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            sa += red[0][w];
            sb += red[1][w];
        }
        const double D = (double)((T)half_hbar * (T)sa);
        const double S = (double)((T)half_vol * (T)sb);
        // a non-finite trial point gives J = inf (objective.py:55-57)
        out[0] = *flag ? INFINITY : D + alpha * S;
        out[1] = D;
        out[2] = S;
        *flag = 0;
    }
}

// ------------------------------------------------------------------ host launchers

template <typename T>
int fused_eval_launch(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, T* L, double* spart,
                      int ns, int* flag, T* grad, double* scalars, cudaStream_t s,
                      cudaEvent_t ev0, cudaEvent_t ev1) {
    GridK<T> gk = make_gridk<T>(dg);
    const int64_t m = grid_n(dg);
    NGF_LAUNCH(k_curv_L<T>, ns, 256, 0, s, gk, a.y, L, spart, flag);
    if (ev0) cudaEventRecord(ev0, s);
    NGF_LAUNCH(k_eval_fused<T>, a.fp.n_cta, kThreads, a.fp.smem_bytes, s, a);
    if (ev1) cudaEventRecord(ev1, s);
    const double vol = dg.spacing[0] * dg.spacing[1] * dg.spacing[2];
    NGF_LAUNCH(k_reduce<T>, blocks_for(3 * m, 256), 256, 0, s, gk, a.fp, a.partial, L, (T)vol,
               (T)alpha, grad);
    NGF_LAUNCH(k_finalize<T>, 1, 256, 0, s, a.dpart, a.fp.n_cta, spart, ns, a.half_hbar, vol / 2,
               alpha, flag, scalars);
    NGF_CHECK_LAUNCH();
    return 0;
}

template <typename T>
int fused_prepare(size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_fused<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    return (int)e;
}

template <typename T>
size_t fused_smem(int wx, int wy, int wz) {
    return fused_smem_bytes<T>(wx, wy, wz);
}

// packed reference terms (gR / nR, 1 / nR) from the exact ones
template <typename T>
__global__ void k_pack_rt(const T* __restrict__ gR, const T* __restrict__ nR, int64_t n,
                          V4T<T>* __restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
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

template <typename T>
int pack_rt(const T* gR, const T* nR, int64_t n, void* out, cudaStream_t s) {
    NGF_LAUNCH(k_pack_rt<T>, blocks_for(n, 256), 256, 0, s, gR, nR, n, (V4T<T>*)out);
    NGF_CHECK_LAUNCH();
    return 0;
}

template int fused_eval_launch<float>(const FusedArgs<float>&, const ngf_grid_t&, double, float*,
                                      double*, int, int*, float*, double*, cudaStream_t,
                                      cudaEvent_t, cudaEvent_t);
template int fused_eval_launch<double>(const FusedArgs<double>&, const ngf_grid_t&, double, double*,
                                       double*, int, int*, double*, double*, cudaStream_t,
                                       cudaEvent_t, cudaEvent_t);
template int fused_prepare<float>(size_t);
template int fused_prepare<double>(size_t);
template size_t fused_smem<float>(int, int, int);
template size_t fused_smem<double>(int, int, int);
template int pack_rt<float>(const float*, const float*, int64_t, void*, cudaStream_t);
template int pack_rt<double>(const double*, const double*, int64_t, void*, cudaStream_t);

}  // namespace ngf
