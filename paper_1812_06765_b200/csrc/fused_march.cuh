// Fused NGF objective/gradient march for sm_100a (the performance path), included by the
// per-variant translation units march_v<n>.cu.
//
// One CTA owns a 32 x TY column of image voxels plus a one-voxel ring
// (E1 = 34 x (TY+2) positions, S slots per thread) and marches a chunk of
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
// ring voxels carry only this tile's contributions; k_post adds the tiles that
// share a deformation node in a fixed order (deterministic, no atomics).
//
// Shared memory has a compile-time layout (SmemL) so every access is one LDS/STS
// with an immediate offset from a per-slot register; x/y differences are plain
// central differences except for the few slots next to a volume face, which use
// the exact one-sided coefficients (warp.py:139-142, :168-175).

#pragma once
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "fused_cfg.cuh"

namespace ngf {

#ifndef NGF_T_PREFETCH
#define NGF_T_PREFETCH 0  // measured slower: 356 vs 340 us at 256^3
#endif

// Per-thread march state.  Slot s owns E1 position P = tid + s * NT for all planes.
template <typename T, typename C>
struct March {
    int P[C::S];        // flat E1 index (E1 = sink for padding slots)
    int P2[C::S];       // index in the zero-padded q layout
    unsigned ij[C::S];  // j * nx + i of the image column (offset inside a plane)
    unsigned flags;     // per slot s, bits 4s..4s+3: in volume (x/y), tile interior, x face, y face
    bool wface;         // some lane of the warp has a slot next to a volume face
    T ylo[C::S][3], yhi[C::S][3];  // P_xy y on the current def-plane pair
    T qz[C::S][3];                 // q_z, plane ring
    T A0[C::S][3], A1[C::S][3];    // z-accumulated ghat for def planes zd, zd+1
    T dT[C::DTS ? 1 : C::S][3][3];  // !DTS: interpolant derivative / h, plane ring
    V4T<T> rt[C::S];               // prefetched reference terms (next B plane)
    int z0, z1, zb, jfirst, jlast, wzlo, cur_zd, cta;
    double dacc;
};

template <typename T, typename C>
__device__ __forceinline__ bool s_vol(const March<T, C>& m, int s) { return (m.flags >> (4 * s)) & 1u; }
template <typename T, typename C>
__device__ __forceinline__ bool s_e0(const March<T, C>& m, int s) { return (m.flags >> (4 * s + 1)) & 1u; }
template <typename T, typename C>
__device__ __forceinline__ bool s_fx(const March<T, C>& m, int s) { return (m.flags >> (4 * s + 2)) & 1u; }
template <typename T, typename C>
__device__ __forceinline__ bool s_fy(const March<T, C>& m, int s) { return (m.flags >> (4 * s + 3)) & 1u; }

template <typename T, typename C>
__device__ __forceinline__ void load_yplane(const FusedArgs<T>& a, const SmemL<T, C>& sm, int P, int zd,
                                            T (&out)[3]) {
    // P_xy y on def plane zd at the slot's image (i, j): x then y (transfer.py:136-142)
    const int ex = P % C::E1X, ey = P / C::E1X;
    const int x0 = sm.colP0[ex], x1 = sm.colP1[ex];
    const int y0 = sm.rowP0[ey], y1 = sm.rowP1[ey];
    const T wx = sm.colPw[ex], wy = sm.rowPw[ey];
    const unsigned mm = (unsigned)(a.ndx * a.ndy * a.ndz);
    // 32-bit element offsets from the one 64-bit base (each load: one add and one wide
    // multiply-add for the address, instead of a 64-bit pointer chain per row and column)
    const unsigned o00 = (unsigned)zd * (unsigned)(a.ndx * a.ndy) + (unsigned)(y0 * a.ndx + x0);
    const unsigned dx = (unsigned)(x1 - x0), dy = (unsigned)((y1 - y0) * a.ndx);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const unsigned o = o00 + (unsigned)k * mm;
        const T X0 = lerp_exact(__ldg(a.y + o), __ldg(a.y + (o + dx)), wx);
        const T X1 = lerp_exact(__ldg(a.y + (o + dy)), __ldg(a.y + (o + dy + dx)), wx);
        out[k] = lerp_exact(X0, X1, wy);
    }
}

// Reduce a completed deformation plane (z-accumulated ghat in `acc`) in x then y over
// the tile's window and write it to the CTA's partial slot zs.
template <typename T, typename C>
__device__ __forceinline__ void flush_plane(const FusedArgs<T>& a, SmemL<T, C>& sm, const int (&P)[C::S],
                                         const T (&acc)[C::S][3], int cta, int zs) {
    const int wx = a.fp.wx, wy = a.fp.wy;
#pragma unroll
    for (int s = 0; s < C::S; ++s) {
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.buf[c][P[s]] = acc[s][c];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < C::E1Y * wx; t += C::NT) {
        const int row = t / wx;
        const int d = t - row * wx;
        const int k0 = sm.xoff[d], k1 = sm.xoff[d + 1];
        T r0 = (T)0, r1 = (T)0, r2 = (T)0;
        for (int k = k0; k < k1; ++k) {
            const int e = row * C::E1X + sm.xcol[k];
            const T w = sm.xw[k];
            r0 = fmaf_t(sm.buf[0][e], w, r0);
            r1 = fmaf_t(sm.buf[1][e], w, r1);
            r2 = fmaf_t(sm.buf[2][e], w, r2);
        }
        sm.Xr[0][row][d] = r0;
        sm.Xr[1][row][d] = r1;
        sm.Xr[2][row][d] = r2;
    }
    __syncthreads();
    const size_t win = (size_t)a.fp.wz * wy * wx;
    T* out = a.partial + (size_t)cta * 3 * win + (size_t)zs * wy * wx;
    for (int t = threadIdx.x; t < wy * wx; t += C::NT) {
        const int dr = t / wx;
        const int d = t - dr * wx;
        const int k0 = sm.yoff[dr], k1 = sm.yoff[dr + 1];
        T r0 = (T)0, r1 = (T)0, r2 = (T)0;
        for (int k = k0; k < k1; ++k) {
            const int row = sm.yrow[k];
            const T w = sm.yw[k];
            r0 = fmaf_t(sm.Xr[0][row][d], w, r0);
            r1 = fmaf_t(sm.Xr[1][row][d], w, r1);
            r2 = fmaf_t(sm.Xr[2][row][d], w, r2);
        }
        out[t] = r0;
        out[win + t] = r1;
        out[2 * win + t] = r2;
    }
}

// One axis of the template cell lookup (warp.py:38-53): t = (p - o) / h with the
// reference's rounding, the hull test, the clamped lower corner and the fraction.
template <typename T, bool POW2>
__device__ __forceinline__ int cell_axis(T p, T o, T h, T ih, T nm1, T hi, bool& inside, T& f) {
    const T d = sub_rn(p, o);
    const T t = POW2 ? mul_rn(d, ih) : div_rn(d, h);
    inside = inside && (t >= (T)0) && (t <= nm1);
    const T fl = fmin_t(fmax_t(floor(t), (T)0), hi);  // NaN -> 0
    f = t - fl;  // exact for inside samples (Sterbenz); outside samples are masked
    return (int)fl;
}

template <int R, typename T, typename C, bool POW2, bool GEN>
__device__ __forceinline__ void fused_step(const FusedArgs<T>& a, SmemL<T, C>& sm, March<T, C>& m,
                                           int p) {
    constexpr int RB = (R + 2) % 3;  // plane p-1
    constexpr int RC = (R + 1) % 3;  // plane p-2
    constexpr int S = C::S;
    const unsigned nxy = (unsigned)a.nx * (unsigned)a.ny;
    const T hx2 = (T)0.5 * a.ihx, hy2 = (T)0.5 * a.ihy;

    // ---------------------------------------------------------------- (A) plane p
    if (p >= 0 && p < a.nz && p <= m.z1) {
        const int zd = sm.zi[p - m.zb][0];
        if (zd != m.cur_zd) {
            const int zd1 = min(zd + 1, a.ndz - 1);
            const bool shift = (zd == m.cur_zd + 1);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (!s_vol(m, s)) continue;
                if (shift) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) m.ylo[s][k] = m.yhi[s][k];
                } else {
                    load_yplane(a, sm, m.P[s], zd, m.ylo[s]);
                }
                load_yplane(a, sm, m.P[s], zd1, m.yhi[s]);
            }
            m.cur_zd = zd;
        }
        const T wz = sm.zt[p - m.zb][6];
        const T wz0 = sm.zt[p - m.zb][7];
        // coordinates and corner offsets of all slots first, so the 8 * S gathers are
        // in flight together
        unsigned off[S];
        T fx[S], fy[S], fz[S];
        bool in[S];
        bool pf[S];  // the template plane after this slot's corner planes exists
#pragma unroll
        for (int s = 0; s < S; ++s) {
            // yhat = Ylo * (1 - w) + Yhi * w, each op rounded (transfer.py:126)
            const T yh0 = add_rn(mul_rn(m.ylo[s][0], wz0), mul_rn(m.yhi[s][0], wz));
            const T yh1 = add_rn(mul_rn(m.ylo[s][1], wz0), mul_rn(m.yhi[s][1], wz));
            const T yh2 = add_rn(mul_rn(m.ylo[s][2], wz0), mul_rn(m.yhi[s][2], wz));
            bool inside = s_vol(m, s);
            const int ix = cell_axis<T, POW2>(yh0, a.ox, a.hx, a.ihx, a.nm1x, a.hix, inside, fx[s]);
            const int iy = cell_axis<T, POW2>(yh1, a.oy, a.hy, a.ihy, a.nm1y, a.hiy, inside, fy[s]);
            const int iz = cell_axis<T, POW2>(yh2, a.oz, a.hz, a.ihz, a.nm1z, a.hiz, inside, fz[s]);
            in[s] = inside;
            pf[s] = iz + 2 < a.nz;
            off[s] = (unsigned)iz * nxy + (unsigned)iy * (unsigned)a.nx + (unsigned)ix;
        }
        T cv[S][8];
        if (GEN) {  // degenerate axes: the +1 corner is the same voxel
            const unsigned sx = a.nx > 1 ? 1u : 0u;
            const unsigned sy = a.ny > 1 ? (unsigned)a.nx : 0u;
            const unsigned sz = a.nz > 1 ? nxy : 0u;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const unsigned o = off[s];
                cv[s][0] = __ldg(a.Tv + o);
                cv[s][1] = __ldg(a.Tv + (o + sx));
                cv[s][2] = __ldg(a.Tv + (o + sy));
                cv[s][3] = __ldg(a.Tv + (o + sy + sx));
                cv[s][4] = __ldg(a.Tv + (o + sz));
                cv[s][5] = __ldg(a.Tv + (o + sz + sx));
                cv[s][6] = __ldg(a.Tv + (o + sz + sy));
                cv[s][7] = __ldg(a.Tv + (o + sz + sy + sx));
            }
        } else {  // one base address per slot, +x corners as immediate offsets
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const T* b = a.Tv + off[s];
                const T* by = b + a.nx;
                const T* bz = b + nxy;
                const T* byz = bz + a.nx;
                cv[s][0] = __ldg(b);
                cv[s][1] = __ldg(b + 1);
                cv[s][2] = __ldg(by);
                cv[s][3] = __ldg(by + 1);
                cv[s][4] = __ldg(bz);
                cv[s][5] = __ldg(bz + 1);
                cv[s][6] = __ldg(byz);
                cv[s][7] = __ldg(byz + 1);
#if NGF_T_PREFETCH
                // the next plane's new corner plane (y advances about one voxel per plane)
                // towards L2, so its first gathers miss L1 but not DRAM
                if (pf[s]) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(bz + nxy));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(byz + nxy));
                }
#endif
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            T W, d0, d1, d2;
            trilinear(a, cv[s], fx[s], fy[s], fz[s], W, d0, d1, d2);
            if (!in[s]) W = d0 = d1 = d2 = (T)0;
            if constexpr (C::DTS) {
                sm.dTs[p & 3][0][m.P[s]] = d0;
                sm.dTs[p & 3][1][m.P[s]] = d1;
                sm.dTs[p & 3][2][m.P[s]] = d2;
            } else {
                m.dT[s][R][0] = d0;
                m.dT[s][R][1] = d1;
                m.dT[s][R][2] = d2;
            }
            sm.Wsm[R][m.P[s]] = W;
        }
    } else {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if constexpr (C::DTS)
                sm.dTs[p & 3][0][m.P[s]] = sm.dTs[p & 3][1][m.P[s]] = sm.dTs[p & 3][2][m.P[s]] = (T)0;
            else
                m.dT[s][R][0] = m.dT[s][R][1] = m.dT[s][R][2] = (T)0;
            sm.Wsm[R][m.P[s]] = (T)0;
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (B) q on plane k = p-1
    T* qxw = sm.qx[p & 1];  // plane p-1 buffer; plane p-2 sits in the other one
    T* qyw = sm.qy[p & 1];
    {
        const int k = p - 1;
        const bool kv = (k >= m.z0) && (k < m.z1);
        const T* zc = sm.zt[max(k - m.zb, 0)];
        const T cmz = zc[0], c0z = zc[1], cpz = zc[2];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            T qxv = (T)0, qyv = (T)0, qzv = (T)0;
            if (kv && s_e0(m, s)) {
                const int P = m.P[s];
                const T w0 = sm.Wsm[RB][P];
                T gx = (sm.Wsm[RB][P + 1] - sm.Wsm[RB][P - 1]) * hx2;
                T gy = (sm.Wsm[RB][P + C::E1X] - sm.Wsm[RB][P - C::E1X]) * hy2;
                if (m.wface) {  // warp holds a slot next to a volume face (rare, uniform)
                    if (s_fx(m, s)) {  // one-sided difference at an x face
                        const T* cg = sm.colG[P % C::E1X];
                        gx = fmaf_t(cg[0], sm.Wsm[RB][P - 1], fmaf_t(cg[1], w0, cg[2] * sm.Wsm[RB][P + 1]));
                    }
                    if (s_fy(m, s)) {
                        const T* rg = sm.rowG[P / C::E1X];
                        gy = fmaf_t(rg[0], sm.Wsm[RB][P - C::E1X],
                                    fmaf_t(rg[1], w0, rg[2] * sm.Wsm[RB][P + C::E1X]));
                    }
                }
                const T gz = fmaf_t(cmz, sm.Wsm[RC][P], fmaf_t(c0z, w0, cpz * sm.Wsm[R][P]));
                ngf_q(a, gx, gy, gz, m.rt[s], qxv, qyv, qzv, m.dacc);
            }
            qxw[m.P2[s]] = qxv;
            qyw[m.P2[s]] = qyv;
            m.qz[s][RB] = qzv;
        }
        // prefetch the reference terms of plane p for the next step's (B)
        if (p >= m.z0 && p < m.z1) {
            const V4T<T>* rp = a.RT + (size_t)p * nxy;
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (s_e0(m, s)) m.rt[s] = ld_rt(rp + m.ij[s]);
        }
    }
    __syncthreads();

    // ---------------------------------------------------------------- (C) s, ghat, z-P^T on j = p-2
    const int j = p - 2;
    if (j < m.jfirst || j > m.jlast) return;  // uniform
    const T* zc = sm.zt[j - m.zb];
    const T gtm = zc[3], gt0 = zc[4], gtp = zc[5], w1 = zc[6], w0 = zc[7];
    const T* qxj = sm.qx[(p & 1) ^ 1];
    const T* qyj = sm.qy[(p & 1) ^ 1];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!s_vol(m, s)) continue;
        const int P2 = m.P2[s];
        T sx = (qxj[P2 - 1] - qxj[P2 + 1]) * hx2;
        T sy = (qyj[P2 - C::E2X] - qyj[P2 + C::E2X]) * hy2;
        if (m.wface) {
            if (s_fx(m, s)) {  // exact transposed face rows (warp.py:168-175)
                const T* ct = sm.colGt[m.P[s] % C::E1X];
                sx = fmaf_t(ct[0], qxj[P2 - 1], fmaf_t(ct[1], qxj[P2], ct[2] * qxj[P2 + 1]));
            }
            if (s_fy(m, s)) {
                const T* rt = sm.rowGt[m.P[s] / C::E1X];
                sy = fmaf_t(rt[0], qyj[P2 - C::E2X], fmaf_t(rt[1], qyj[P2], rt[2] * qyj[P2 + C::E2X]));
            }
        }
        T sv = add_rn(sx, sy);  // no contraction (the packed march adds the same way)
        sv = fmaf_t(gtm, m.qz[s][R], fmaf_t(gt0, m.qz[s][RC], fmaf_t(gtp, m.qz[s][RB], sv)));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T g = sv * (C::DTS ? sm.dTs[j & 3][c][m.P[s]] : m.dT[s][RC][c]);
            m.A0[s][c] = fmaf_t(w0, g, m.A0[s][c]);
            m.A1[s][c] = fmaf_t(w1, g, m.A1[s][c]);
        }
    }
    // def plane zdj is complete when the next image plane maps to a later pair.  The map
    // can advance by 2 (w1 rounds to just below 1 when the grids nearly coincide), in
    // which case zdj + 1 is complete as well.
    const int zdj = sm.zi[j - m.zb][0];
    const int step = (j == m.jlast) ? 2 : sm.zi[j - m.zb][1];
    if (step >= 1) {
        flush_plane<T, C>(a, sm, m.P, m.A0, m.cta, zdj - m.wzlo);
        if (step >= 2) {
            if (zdj + 1 <= a.ndz - 1) {
                __syncthreads();
                flush_plane<T, C>(a, sm, m.P, m.A1, m.cta, zdj + 1 - m.wzlo);
            }
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < 3; ++c) m.A0[s][c] = m.A1[s][c] = (T)0;
        } else {
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    m.A0[s][c] = m.A1[s][c];
                    m.A1[s][c] = (T)0;
                }
        }
    }
}

// CTA geometry of the march
struct CtaGeo {
    int tx, ty, tz, x0, y0, z0, z1, zb, jfirst, jlast, wzlo;
};

template <typename T, typename C>
__device__ __forceinline__ CtaGeo cta_geo(const FusedArgs<T>& a) {
    const FusedPlan& fp = a.fp;
    CtaGeo g;
    const int cta = blockIdx.x;
    g.tx = cta % fp.ntx;
    g.ty = (cta / fp.ntx) % fp.nty;
    g.tz = cta / (fp.ntx * fp.nty);
    g.x0 = g.tx * C::TX;
    g.y0 = g.ty * C::TY;
    g.z0 = fp.zb_tab[g.tz];
    g.z1 = fp.zb_tab[g.tz + 1];
    g.zb = g.z0 - 1;  // first plane of the z tables
    g.jfirst = max(g.z0 - 1, 0);
    g.jlast = min(g.z1, a.nz - 1);
    g.wzlo = fp.win_z[g.tz];
    return g;
}

// per-CTA shared tables: face coefficients, P weights, z tables, zeroed q rings, P^T CSR
template <typename T, typename C>
__device__ __forceinline__ void cta_tables(const FusedArgs<T>& a, SmemL<T, C>& sm, const CtaGeo& g) {
    const FusedPlan& fp = a.fp;
    const int tid = threadIdx.x;
    for (int e = tid; e < C::E1X; e += C::NT) {
        const int i = g.x0 - 1 + e;
        fd_coef<T>(i, a.nx, a.ihx, sm.colG[e][0], sm.colG[e][1], sm.colG[e][2]);
        fdt_coef<T>(i, a.nx, a.ihx, sm.colGt[e][0], sm.colGt[e][1], sm.colGt[e][2]);
        const bool in = i >= 0 && i < a.nx;
        const int i0 = in ? a.i0x[i] : 0;
        sm.colP0[e] = i0;
        sm.colP1[e] = min(i0 + 1, a.ndx - 1);
        sm.colPw[e] = in ? a.w1x[i] : (T)0;
    }
    for (int e = tid; e < C::E1Y; e += C::NT) {
        const int jj = g.y0 - 1 + e;
        fd_coef<T>(jj, a.ny, a.ihy, sm.rowG[e][0], sm.rowG[e][1], sm.rowG[e][2]);
        fdt_coef<T>(jj, a.ny, a.ihy, sm.rowGt[e][0], sm.rowGt[e][1], sm.rowGt[e][2]);
        const bool in = jj >= 0 && jj < a.ny;
        const int i0 = in ? a.i0y[jj] : 0;
        sm.rowP0[e] = i0;
        sm.rowP1[e] = min(i0 + 1, a.ndy - 1);
        sm.rowPw[e] = in ? a.w1y[jj] : (T)0;
    }
    for (int t = tid; t < g.z1 + 2 - g.zb; t += C::NT) {
        // z tables for planes zb .. z1+1 (coefficients of warp.py:130-176 along z, P's w1)
        const int z = g.zb + t;
        T* zc = sm.zt[t];
        fd_coef<T>(z, a.nz, a.ihz, zc[0], zc[1], zc[2]);
        fdt_coef<T>(z, a.nz, a.ihz, zc[3], zc[4], zc[5]);
        const bool in = z >= 0 && z < a.nz;
        const T w1 = in ? a.w1z[z] : (T)0;
        zc[6] = w1;
        zc[7] = sub_rn((T)1, w1);
        sm.zi[t][0] = in ? a.i0z[z] : 0;
        sm.zi[t][1] = (in && z + 1 < a.nz) ? a.i0z[z + 1] - a.i0z[z] : 2;
    }
    for (int t = tid; t < 2 * C::E2; t += C::NT) {
        (&sm.qx[0][0])[t] = (T)0;
        (&sm.qy[0][0])[t] = (T)0;
    }
    // this tile's CSR of the transposed 1-D interpolation (host-built, ascending E1
    // index per window entry: the reference's gather order, transfer.py:89-96)
    const int sxs = fp.wx + 1 + 2 * C::E1X, sys = fp.wy + 1 + 2 * C::E1Y;
    const int32_t* gx = fp.xcsr + (size_t)g.tx * sxs;
    const int32_t* gy = fp.ycsr + (size_t)g.ty * sys;
    const T* wxg = (const T*)fp.xcw + (size_t)g.tx * 2 * C::E1X;
    const T* wyg = (const T*)fp.ycw + (size_t)g.ty * 2 * C::E1Y;
    for (int t = tid; t < fp.wx + 1; t += C::NT) sm.xoff[t] = gx[t];
    for (int t = tid; t < 2 * C::E1X; t += C::NT) {
        sm.xcol[t] = gx[fp.wx + 1 + t];
        sm.xw[t] = wxg[t];
    }
    for (int t = tid; t < fp.wy + 1; t += C::NT) sm.yoff[t] = gy[t];
    for (int t = tid; t < 2 * C::E1Y; t += C::NT) {
        sm.yrow[t] = gy[fp.wy + 1 + t];
        sm.yw[t] = wyg[t];
    }
}

// Slot s of a thread owns E1 position tid + s * NT for all planes: its E1 index (padding
// slots -> the sink entry E1), zero-padded q index, image column offset and flag bits
// (in volume (x/y), tile interior, x face, y face).
template <typename T, typename C>
__device__ __forceinline__ void slot_geom(const FusedArgs<T>& a, const CtaGeo& g, int s, int& Pout, int& P2out,
                                          unsigned& ij, unsigned& flags) {
    const T hx2 = (T)0.5 * a.ihx, hy2 = (T)0.5 * a.ihy;
    // slot q -> E1 position: the tile interior first, row by row (each warp's lanes cover
    // one 32-wide interior row, so (B), which only runs on the interior, is warp-uniform),
    // then the ring (top row, bottom row, left/right columns), then padding
    const int q = threadIdx.x + s * C::NT;
    constexpr int NI = C::TX * C::TY;
    const bool ok = q < C::E1;
    int ex = 0, ey = 0;
    if (q < NI) {
        ex = q % C::TX + 1;
        ey = q / C::TX + 1;
    } else if (q < NI + C::E1X) {
        ex = q - NI;
    } else if (q < NI + 2 * C::E1X) {
        ex = q - NI - C::E1X;
        ey = C::E1Y - 1;
    } else if (ok) {
        const int rr = q - NI - 2 * C::E1X;
        ey = 1 + rr / 2;
        ex = (rr & 1) ? C::E1X - 1 : 0;
    }
    const int Pc = ok ? ey * C::E1X + ex : C::E1;
    if (!ok) ex = ey = 0;
    const int i = g.x0 - 1 + ex, jj = g.y0 - 1 + ey;
    const bool vol = ok && i >= 0 && i < a.nx && jj >= 0 && jj < a.ny;
    const bool e0 = vol && ex >= 1 && ex <= C::TX && ey >= 1 && ey <= C::TY;
    // a slot needs the exact face coefficients where G or G^T differ from central
    T cm, c0, cp, gm, g0, gp;
    fd_coef<T>(i, a.nx, a.ihx, cm, c0, cp);
    fdt_coef<T>(i, a.nx, a.ihx, gm, g0, gp);
    const bool fx = !(cm == -hx2 && c0 == (T)0 && cp == hx2 && gm == hx2 && g0 == (T)0 && gp == -hx2);
    fd_coef<T>(jj, a.ny, a.ihy, cm, c0, cp);
    fdt_coef<T>(jj, a.ny, a.ihy, gm, g0, gp);
    const bool fy = !(cm == -hy2 && c0 == (T)0 && cp == hy2 && gm == hy2 && g0 == (T)0 && gp == -hy2);
    Pout = Pc;
    P2out = ok ? (ey + 1) * C::E2X + ex + 1 : 0;  // padding slots write 0 into the pad ring
    ij = vol ? (unsigned)(jj * a.nx + i) : 0u;
    flags = (vol ? 1u : 0u) | (e0 ? 2u : 0u) | (vol && fx ? 4u : 0u) | (vol && fy ? 8u : 0u);
}

// the CTA's D partial (fixed order: warp tree, then warps in order)
template <typename T, typename C>
__device__ __forceinline__ void cta_dpart(const FusedArgs<T>& a, SmemL<T, C>& sm, double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sacc = 0.0;
        for (int w = 0; w < C::NT / 32; ++w) sacc += sm.red[w];
        a.dpart[blockIdx.x] = sacc;
    }
}

template <typename T, typename C, bool POW2, bool GEN>
__global__ void __launch_bounds__(C::NT, C::MINB) k_eval_fused(const __grid_constant__ FusedArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemL<T, C>& sm = *reinterpret_cast<SmemL<T, C>*>(smem_raw);
    constexpr int S = C::S;
    const CtaGeo g = cta_geo<T, C>(a);
    March<T, C> m;
    m.cta = blockIdx.x;
    m.z0 = g.z0;
    m.z1 = g.z1;
    m.zb = g.zb;
    m.jfirst = g.jfirst;
    m.jlast = g.jlast;
    m.wzlo = g.wzlo;
    m.cur_zd = -1000;
    m.dacc = 0.0;
    cta_tables<T, C>(a, sm, g);

    // ---- slot positions (fixed for all planes)
    m.flags = 0u;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        unsigned fl;
        slot_geom<T, C>(a, g, s, m.P[s], m.P2[s], m.ij[s], fl);
        m.flags |= fl << (4 * s);
#pragma unroll
        for (int r = 0; r < 3; ++r) m.qz[s][r] = (T)0;
        if constexpr (C::DTS) {
#pragma unroll
            for (int r = 0; r < 4; ++r) sm.dTs[r][0][m.P[s]] = sm.dTs[r][1][m.P[s]] = sm.dTs[r][2][m.P[s]] = (T)0;
        } else {
#pragma unroll
            for (int r = 0; r < 3; ++r) m.dT[s][r][0] = m.dT[s][r][1] = m.dT[s][r][2] = (T)0;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            m.ylo[s][c] = m.yhi[s][c] = (T)0;
            m.A0[s][c] = m.A1[s][c] = (T)0;
        }
        m.rt[s] = V4T<T>{};
    }
    m.wface = __any_sync(0xffffffffu, (m.flags & 0xCCCCCCCCu) != 0u);
    __syncthreads();
    // reference terms of the first interior plane
    if (m.z0 < m.z1) {
        const V4T<T>* rp = a.RT + (size_t)m.z0 * a.nx * a.ny;
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (s_e0(m, s)) m.rt[s] = ld_rt(rp + m.ij[s]);
    }

    // planes p = z0-1 .. z1+2: (A) on p, (B) on p-1, (C) on p-2
    const int pstart = m.z0 - 1;
    const int nsteps = (m.z1 + 2) - pstart + 1;
    for (int b = 0; b < nsteps; b += 3) {
        fused_step<0, T, C, POW2, GEN>(a, sm, m, pstart + b);
        if (b + 1 < nsteps) fused_step<1, T, C, POW2, GEN>(a, sm, m, pstart + b + 1);
        if (b + 2 < nsteps) fused_step<2, T, C, POW2, GEN>(a, sm, m, pstart + b + 2);
    }
    cta_dpart<T, C>(a, sm, m.dacc);
}

#include "fused_pair.cuh"

template <typename K>
static cudaError_t smem_attr(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// The dynamic shared memory limit is a per-kernel attribute shared by every level and
// thread: it is only ever raised (levels of different sizes are created concurrently by
// registrations on other streams, and a lowered limit would fail their launches).
template <typename T, typename C>
int march_prepare(size_t smem) {
    static std::mutex mu;
    static size_t granted = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (smem <= granted) return 0;
    cudaError_t e = smem_attr(k_eval_fused<T, C, true, false>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, false, false>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, true, true>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, false, true>, smem);
    if constexpr (kPaired<T, C>) {
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, true, false>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, false, false>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, true, true>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, false, true>, smem);
    }
    if (e == cudaSuccess) granted = smem;
    return (int)e;
}

template <typename T, typename C>
void march_launch(const FusedArgs<T>& a, cudaStream_t s) {
    const bool pow2 = a.pow2x && a.pow2y && a.pow2z;
    const bool gen = a.nx < 2 || a.ny < 2 || a.nz < 2;  // a degenerate image axis
    if constexpr (kPaired<T, C>) {
        if (a.fp.packed) {
            if (pow2 && !gen)
                NGF_LAUNCH((k_eval_pair<C, true, false>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
            else if (!gen)
                NGF_LAUNCH((k_eval_pair<C, false, false>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
            else if (pow2)
                NGF_LAUNCH((k_eval_pair<C, true, true>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
            else
                NGF_LAUNCH((k_eval_pair<C, false, true>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
            return;
        }
    }
    if (pow2 && !gen)
        NGF_LAUNCH((k_eval_fused<T, C, true, false>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
    else if (!gen)
        NGF_LAUNCH((k_eval_fused<T, C, false, false>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
    else if (pow2)
        NGF_LAUNCH((k_eval_fused<T, C, true, true>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
    else
        NGF_LAUNCH((k_eval_fused<T, C, false, true>), a.fp.n_cta, C::NT, a.fp.smem_bytes, s, a);
}


}  // namespace ngf
