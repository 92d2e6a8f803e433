// Fused NGF objective/gradient evaluation for sm_100a (the performance path).
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

#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "eval_fused.cuh"
#include "fused_impl.cuh"

namespace ngf {


// Tile / launch configuration of one kernel variant.
template <int TY_, int NT_, int MINB_, bool DTS_ = false>
struct Cfg {
    static constexpr int TX = 32, TY = TY_, NT = NT_, MINB = MINB_;
    static constexpr bool DTS = DTS_;  // interpolant derivative ring in shared memory (frees 9 S registers)
    static constexpr int E1X = TX + 2, E1Y = TY + 2, E1 = E1X * E1Y;
    static constexpr int S = (E1 + NT - 1) / NT;
    static constexpr int E2X = TX + 4, E2Y = TY + 4, E2 = E2X * E2Y;
    // P^T window bounds: the ring widens a tile by 2 voxels, +1 for the upper node, +1 where
    // the index map advances by 2 (w1 rounding to just below 1 when grids nearly coincide)
    static constexpr int WXMAX = E1X + 2, WYMAX = E1Y + 2;
};

template <typename T>
__host__ __device__ __forceinline__ void fd_coef(int i, int n, T ih, T& cm, T& c0, T& cp) {
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
__host__ __device__ __forceinline__ void fdt_coef(int i, int n, T ih, T& gm, T& g0, T& gp) {
    T a, b, c;
    fd_coef<T>(i - 1, n, ih, a, b, c);
    gm = c;
    fd_coef<T>(i, n, ih, a, b, c);
    g0 = b;
    fd_coef<T>(i + 1, n, ih, a, b, c);
    gp = a;
}

// Compile-time shared memory layout.
template <typename T, typename C>
struct SmemL {
    T Wsm[3][C::E1 + 1];        // W ring (planes p-2, p-1, p); [E1] = padding-slot sink
    T qx[2][C::E2], qy[2][C::E2];  // q_x, q_y of planes p-1 (written) / p-2 (read), zero-padded
    T buf[3][C::E1 + 1];        // completed deformation plane (z-reduced ghat)
    T dTs[C::DTS ? 4 : 1][3][C::DTS ? C::E1 + 1 : 1];  // DTS: interpolant derivative / h,
                                // [plane & 3][axis][E1 position] (4 slots: (C) of step p-1 may still read plane p-3)
    T Xr[3][C::E1Y][C::WXMAX];  // x-reduced
    T colG[C::E1X][3], colGt[C::E1X][3], rowG[C::E1Y][3], rowGt[C::E1Y][3];  // face coefficients
    T colPw[C::E1X], rowPw[C::E1Y];  // P weights
    T xw[2 * C::E1X], yw[2 * C::E1Y];  // CSR weights
    T zt[kCzMax + 4][8];        // per plane: G (cm,c0,cp), G^T (gm,g0,gp), w1z, 1-w1z
    int zi[kCzMax + 4][2];      // per plane: i0z, advance of i0z to the next plane
    int colP0[C::E1X], colP1[C::E1X], rowP0[C::E1Y], rowP1[C::E1Y];
    int xoff[C::WXMAX + 1], xcol[2 * C::E1X], yoff[C::WYMAX + 1], yrow[2 * C::E1Y];
    double red[C::NT / 32];
};

template <typename T, typename C>
__host__ __device__ inline size_t smem_bytes_cfg(int wx, int wy) {
    if (wx > C::WXMAX || wy > C::WYMAX) return size_t(1) << 30;  // cannot happen for valid plans
    return sizeof(SmemL<T, C>);
}

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
    const unsigned plane = (unsigned)zd * (unsigned)(a.ndx * a.ndy);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T* yc = a.y + (k * mm + plane);
        const T* r0 = yc + y0 * a.ndx;
        const T* r1 = yc + y1 * a.ndx;
        const T X0 = lerp_exact(__ldg(r0 + x0), __ldg(r0 + x1), wx);
        const T X1 = lerp_exact(__ldg(r1 + x0), __ldg(r1 + x1), wx);
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

// ------------------------------------------------------------------ reduce + curvature

// One kernel after the march: grad = grad D (fixed-order sum of the covering tiles'
// partials) + alpha * vol * L^T L u (curvature.py:74-81), the per-block partial sums of
// (L u)^2, and -- in the last block to finish -- the fixed-order totals J, D, S.
// Grid: x/y tiles of 32 x 8 deformation nodes, blockIdx.z = comp * nchunk + z chunk.
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
constexpr int kPostKZ = 4;
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
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    const int bid = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const int comp = blockIdx.z / p.nchunk, chunk = blockIdx.z - comp * p.nchunk;
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
        last = atomicAdd(p.flag + 1, 1) == nblk - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        post_finalize<T>(p, nblk);
    }
}

// ------------------------------------------------------------------ host launchers

// Kernel variants: tile rows TY, threads per CTA, minimum resident CTAs per SM, derivative
// ring in shared memory (tools/sweep.py).  f32 default: 32 x 16 tiles of 320 threads with
// the ring in shared memory (96 registers, 2 CTAs = 20 warps per SM, ring overhead 1.2);
// 32 x 12 / 256 threads keeps the ring in registers (128 registers, 16 warps per SM) and
// wins when its CTA count fills the waves better.  f64 uses one slot per thread (32 x 16
// tiles of 640 threads or 32 x 12 of 512, one CTA per SM): its march state per slot is
// twice as large, and the two-slot 32 x 20 shape (variant 0) spills 1.3 KB per thread
// (942 us vs 638 us at 256^3).
using V0 = Cfg<20, 256, 2>;
using V1 = Cfg<12, 256, 2>;
using V2 = Cfg<16, 320, 2, true>;
using V3 = Cfg<18, 352, 2, true>;
// f64 shapes: one slot per thread (a slot's f64 march state needs about twice the registers)
using V4 = Cfg<12, 512, 1, true>;
using V5 = Cfg<16, 640, 1, true>;
constexpr int kNumVariants = 6;

void fused_variant_geom(int v, int* ty, int* nt) {
    switch (v) {
        case 1: *ty = V1::TY; *nt = V1::NT; return;
        case 2: *ty = V2::TY; *nt = V2::NT; return;
        case 3: *ty = V3::TY; *nt = V3::NT; return;
        case 4: *ty = V4::TY; *nt = V4::NT; return;
        case 5: *ty = V5::TY; *nt = V5::NT; return;
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
        default: return smem_bytes_cfg<T, V0>(wx, wy);
    }
}

template <typename K>
static cudaError_t smem_attr(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <typename T, typename C>
static int prep(size_t smem) {
    cudaError_t e = smem_attr(k_eval_fused<T, C, true, false>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, false, false>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, true, true>, smem);
    if (e == cudaSuccess) e = smem_attr(k_eval_fused<T, C, false, true>, smem);
    if constexpr (std::is_same<T, float>::value && C::S == 2) {
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, true, false>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, false, false>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, true, true>, smem);
        if (e == cudaSuccess) e = smem_attr(k_eval_pair<C, false, true>, smem);
    }
    return (int)e;
}

template <typename T, typename C>
static void launch(const FusedArgs<T>& a, cudaStream_t s) {
    const bool pow2 = a.pow2x && a.pow2y && a.pow2z;
    const bool gen = a.nx < 2 || a.ny < 2 || a.nz < 2;  // a degenerate image axis
    if constexpr (std::is_same<T, float>::value && C::S == 2) {
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

template <>
int fused_prepare<float>(int v, size_t smem) {
    switch (v) {
        case 1: return prep<float, V1>(smem);
        case 2: return prep<float, V2>(smem);
        case 3: return prep<float, V3>(smem);
        default: return prep<float, V0>(smem);
    }
}

template <>
int fused_prepare<double>(int v, size_t smem) {
    switch (v) {
        case 4: return prep<double, V4>(smem);
        case 5: return prep<double, V5>(smem);
        default: return prep<double, V0>(smem);
    }
}

template <typename T>
static void launch_variant(const FusedArgs<T>& a, cudaStream_t s);

template <>
void launch_variant<float>(const FusedArgs<float>& a, cudaStream_t s) {
    switch (a.fp.variant) {
        case 1: launch<float, V1>(a, s); return;
        case 2: launch<float, V2>(a, s); return;
        case 3: launch<float, V3>(a, s); return;
        default: launch<float, V0>(a, s); return;
    }
}

template <>
void launch_variant<double>(const FusedArgs<double>& a, cudaStream_t s) {
    switch (a.fp.variant) {
        case 4: launch<double, V4>(a, s); return;
        case 5: launch<double, V5>(a, s); return;
        default: launch<double, V0>(a, s); return;
    }
}

template <typename T>
int fused_eval_launch(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int ns,
                      int* flag, T* grad, double* scalars, cudaStream_t s, cudaEvent_t ev0,
                      cudaEvent_t ev1, int part) {
    // part 0: full evaluation; 1: NGF partial of the level's z-slab (grad <- grad D_slab,
    // scalars <- D_slab); 2: add curvature to an all-reduced (grad D, D) in place
    const int nchunk = (int)((dg.dims[2] + kPostKZ - 1) / kPostKZ);
    const dim3 cgrid((dg.dims[0] + 31) / 32, (dg.dims[1] + 7) / 8, 3 * nchunk);
    const int nsb = (int)(cgrid.x * cgrid.y * cgrid.z);
    if (nsb > ns) return NGF_EARG;
    const double vol = dg.spacing[0] * dg.spacing[1] * dg.spacing[2];
    if (part != 2) {
        if (ev0) cudaEventRecord(ev0, s);
        launch_variant<T>(a, s);
        if (ev1) cudaEventRecord(ev1, s);
    }
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
    p.ihx2 = (T)1 / (p.g.hx * p.g.hx);
    p.ihy2 = (T)1 / (p.g.hy * p.g.hy);
    p.ihz2 = (T)1 / (p.g.hz * p.g.hz);
    if (part == 2) {
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


template int fused_eval_launch<float>(const FusedArgs<float>&, const ngf_grid_t&, double, double*, int,
                                      int*, float*, double*, cudaStream_t, cudaEvent_t, cudaEvent_t,
                                      int);
template int fused_eval_launch<double>(const FusedArgs<double>&, const ngf_grid_t&, double, double*,
                                       int, int*, double*, double*, cudaStream_t, cudaEvent_t,
                                       cudaEvent_t, int);
template size_t fused_smem<float>(int, int, int);
template size_t fused_smem<double>(int, int, int);
template int pack_rt<float>(const float*, const float*, int64_t, void*, cudaStream_t);
template int pack_rt<double>(const double*, const double*, int64_t, void*, cudaStream_t);

}  // namespace ngf
