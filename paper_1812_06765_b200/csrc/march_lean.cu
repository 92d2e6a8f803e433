// Lean fused NGF objective/gradient march (f32, sm_100a).
//
// The same pipeline as fused_march.cuh -- per image plane p of a z chunk:
//   (A) yhat = P y bit-exactly (transfer.py:117-148, so the inside/floor decisions of
//       warp.py:32-53 match the reference), the 8 template corners, W (warp.py:64-90)
//       and the interpolant derivative (warp.py:93-127);
//   (B) grad W (warp.py:130-143), the NGF ratio, the distance term and q (ngf.py:70-112)
//       on plane p-1;
//   (C) G^T q (warp.py:159-184) times the derivative on plane p-2, accumulated along z
//       into the two deformation planes it interpolates (transfer.py:151-192, z first);
// -- re-laid out so that a step costs about half the instructions of the classic march:
//   * one position per thread (no slot loops or per-slot flag decoding): 14 row warps,
//     2 ring-row warps and 1 ring-column warp cover the 34 x 16 tile + ring exactly, and
//     the tile is 32 wide in x, so a 256-wide level is 8 tiles with no padding;
//   * ONE __syncthreads per plane: W, q_x and q_y live in triple-buffered shared planes
//     (a warp may run one step ahead of the slowest one without overwriting what it
//     reads); the z neighbours of W and q and the derivative ring stay in registers;
//   * template reads outside the image hull are redirected to a zero pad after the
//     volume (one select instead of masking W and three derivatives), and the inside
//     test compares the float bit patterns of t and n-1 (0 <= t <= n-1 for t >= +0);
//   * the x / y P^T reduction of a completed deformation plane is staggered over the next
//     two steps (x pass after the next barrier, y pass after the one after), with
//     compile-time entry counts per window output and no integer division, and the
//     1/h derivative scale is applied once per deformation node there;
//   * the distance term accumulates in f32 per thread (<= 100 planes), reduced in f64
//     per CTA.
// Determinism: every sum has a fixed order; no atomics.

#include <mutex>

#include "fused_cfg.cuh"
#include "march_lean.cuh"

namespace ngf {
namespace lean {

struct Smem {
    float W[3][kE1Y][kE1X];         // W of planes p-2, p-1, p (ring by plane index mod 3)
    float Qx[3][kE1Y][kE1X + 2];    // q_x, one zero column each side
    float Qy[3][kE1Y + 2][kE1X];    // q_y, one zero row each side
    float Fb[3][kE1Y][kE1X];        // completed deformation plane (z-reduced ghat / h)
    float dTs[3][3][kE1Y * kE1X];   // interpolant derivative (times h) of planes p-2, p-1, p
    float Xr[3][kE1Y][kWXM];        // x-reduced
    float zt[kCzMax + 4][8];        // per plane: G (cm, c0, cp), G^T (gm, g0, gp), w1z, 1 - w1z
    int zi[kCzMax + 4][4];          // per plane: i0z, advance of i0z to the next plane, face flag
    int2 xl[kWXM][kKMax];           // x pass: (E1 column, weight bits) per window output
    int2 yl[kWYM][kKMax];           // y pass: (E1 row, weight bits)
    float colG[kE1X][3], colGt[kE1X][3], rowG[kE1Y][3], rowGt[kE1Y][3];
    int colP0[kE1X], colP1[kE1X], rowP0[kE1Y], rowP1[kE1Y];
    float colPw[kE1X], rowPw[kE1Y];
    double red[kWarps];
};

__device__ __forceinline__ float lerp_x(float a0, float a1, float w, float w0) {
    // a0 * (1 - w) + a1 * w, each op correctly rounded (transfer.py:126)
    return __fadd_rn(__fmul_rn(a0, w0), __fmul_rn(a1, w));
}

template <int KX, int KY>
struct Lean {
    const FusedArgs<float>& a;
    Smem& sm;
    // position of this thread in the tile
    int ex, ey, P;  // E1 column / row, flat index ey * kE1X + ex
    int x, yy;
    bool vol, inter, fx, fy;
    bool wface_b, wface_c;  // warp holds a face position (B: interior, C: any)
    unsigned ij;            // yy * nx + x (reference-term offset inside a plane)
    // chunk
    int cta, z0, z1, zb, jfirst, jlast, wzlo;
    // flush pass assignment, bytes (x pass row, x pass column, y pass row, y pass column),
    // 0xff = none
    unsigned fa;
    // march state
    int cur_zd;
    float ylo[3], yhi[3];
    float qz[3];
    float A0[3], A1[3];
    float4 rt;
    float dacc;
    int xz, yz;  // pending x / y pass (window slot), -1 none

    __device__ __forceinline__ Lean(const FusedArgs<float>& a_, Smem& sm_) : a(a_), sm(sm_) {}

    __device__ __forceinline__ void load_yplane(int zd, float (&out)[3]) const {
        // P_xy y on def plane zd at this position's image (x, y): x then y (transfer.py:136-142)
        const int x0 = sm.colP0[ex], x1 = sm.colP1[ex];
        const int y0 = sm.rowP0[ey], y1 = sm.rowP1[ey];
        const float wx = sm.colPw[ex], wy = sm.rowPw[ey];
        const float wx0 = __fsub_rn(1.0f, wx), wy0 = __fsub_rn(1.0f, wy);
        const unsigned mm = (unsigned)(a.ndx * a.ndy * a.ndz);
        const unsigned o00 = (unsigned)zd * (unsigned)(a.ndx * a.ndy) + (unsigned)(y0 * a.ndx + x0);
        const unsigned dx = (unsigned)(x1 - x0), dy = (unsigned)((y1 - y0) * a.ndx);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const unsigned o = o00 + (unsigned)k * mm;
            const float X0 = lerp_x(__ldg(a.y + o), __ldg(a.y + (o + dx)), wx, wx0);
            const float X1 = lerp_x(__ldg(a.y + (o + dy)), __ldg(a.y + (o + dy + dx)), wx, wx0);
            out[k] = lerp_x(X0, X1, wy, wy0);
        }
    }

    // one axis of the cell lookup (warp.py:38-53): t = (p - o) / h (power-of-two h: an
    // exact multiply), hull test 0 <= t <= n - 1, lower corner min(floor t, n - 2), fraction
    __device__ __forceinline__ int cell(float p, float o, float ih, float nm1, float hi, bool& in, float& f) const {
        const float t = __fmul_rn(__fsub_rn(p, o), ih);
        in = in && (__float_as_uint(t) <= __float_as_uint(nm1));  // NaN and t < 0 (incl. -0) fail
        const float fl = fminf(floorf(t), hi);
        f = t - fl;
        return (int)fl;
    }

    // x pass of a completed deformation plane: Fb -> Xr (fixed entry order per output)
    __device__ __forceinline__ void xpass() {
        const int xr_r = fa & 0xff, xr_d = (fa >> 8) & 0xff;
        if (xr_r != 0xff) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int k = 0; k < KX; ++k) {
                const int2 e = sm.xl[xr_d][k];
                const float w = __int_as_float(e.y);
                s0 = fmaf(w, sm.Fb[0][xr_r][e.x], s0);
                s1 = fmaf(w, sm.Fb[1][xr_r][e.x], s1);
                s2 = fmaf(w, sm.Fb[2][xr_r][e.x], s2);
            }
            sm.Xr[0][xr_r][xr_d] = s0;
            sm.Xr[1][xr_r][xr_d] = s1;
            sm.Xr[2][xr_r][xr_d] = s2;
        }
    }

    // y pass: Xr -> the CTA's window partial of deformation plane slot zs (1/h applied)
    __device__ __forceinline__ void ypass(int zs) {
        const int yp_dy = (fa >> 16) & 0xff, yp_d = fa >> 24;
        if (yp_dy != 0xff) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int k = 0; k < KY; ++k) {
                const int2 e = sm.yl[yp_dy][k];
                const float w = __int_as_float(e.y);
                s0 = fmaf(w, sm.Xr[0][e.x][yp_d], s0);
                s1 = fmaf(w, sm.Xr[1][e.x][yp_d], s1);
                s2 = fmaf(w, sm.Xr[2][e.x][yp_d], s2);
            }
            const int wx = a.fp.wx, wy = a.fp.wy;
            const size_t win = (size_t)a.fp.wz * wy * wx;
            float* out = a.partial + (size_t)cta * 3 * win + (size_t)zs * wy * wx + yp_dy * wx + yp_d;
            out[0] = s0 * a.ihx;
            out[win] = s1 * a.ihy;
            out[2 * win] = s2 * a.ihz;
        }
    }

    __device__ __forceinline__ void put_flush(const float (&acc)[3]) {
        float* b = &sm.Fb[0][0][0] + P;
        b[0] = acc[0];
        b[kE1Y * kE1X] = acc[1];
        b[2 * kE1Y * kE1X] = acc[2];
    }

    template <int R>
    __device__ __forceinline__ void step(int p) {
        constexpr int RB = (R + 2) % 3;  // plane p-1
        constexpr int RC = (R + 1) % 3;  // plane p-2
        const float hx2 = 0.5f * a.ihx, hy2 = 0.5f * a.ihy, hz2 = 0.5f * a.ihz;

        // ------------------------------------------------------------- (A) plane p
        float W = 0.f, d0 = 0.f, d1 = 0.f, d2 = 0.f;
        if (p >= 0 && p < a.nz && p <= z1) {
            const int t = p - zb;
            const int zd = sm.zi[t][0];
            if (zd != cur_zd) {  // CTA-uniform
                const int zd1 = min(zd + 1, a.ndz - 1);
                if (zd == cur_zd + 1) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) ylo[k] = yhi[k];
                } else {
                    load_yplane(zd, ylo);
                }
                load_yplane(zd1, yhi);
                cur_zd = zd;
            }
            const float wz = sm.zt[t][6], wz0 = sm.zt[t][7];
            const float yh0 = __fadd_rn(__fmul_rn(ylo[0], wz0), __fmul_rn(yhi[0], wz));
            const float yh1 = __fadd_rn(__fmul_rn(ylo[1], wz0), __fmul_rn(yhi[1], wz));
            const float yh2 = __fadd_rn(__fmul_rn(ylo[2], wz0), __fmul_rn(yhi[2], wz));
            bool in = vol;
            float fx_, fy_, fz_;
            const int ix = cell(yh0, a.ox, a.ihx, a.nm1x, a.hix, in, fx_);
            const int iy = cell(yh1, a.oy, a.ihy, a.nm1y, a.hiy, in, fy_);
            const int iz = cell(yh2, a.oz, a.ihz, a.nm1z, a.hiz, in, fz_);
            const unsigned nx = (unsigned)a.nx, nxy = nx * (unsigned)a.ny;
            const unsigned off = in ? (unsigned)iz * nxy + (unsigned)iy * nx + (unsigned)ix : a.fp.pad_off;
            const float* b = a.Tv + off;
            const float* by = b + nx;
            const float* bz = b + nxy;
            const float* byz = bz + nx;
            const float c0 = __ldg(b), c1 = __ldg(b + 1), c2 = __ldg(by), c3 = __ldg(by + 1);
            const float c4 = __ldg(bz), c5 = __ldg(bz + 1), c6 = __ldg(byz), c7 = __ldg(byz + 1);
            // trilinear value and derivative (times h) in lerp form (warp.py:79-85, :111-120)
            const float e00 = c1 - c0, e10 = c3 - c2, e01 = c5 - c4, e11 = c7 - c6;
            const float a00 = fmaf(fx_, e00, c0), a10 = fmaf(fx_, e10, c2);
            const float a01 = fmaf(fx_, e01, c4), a11 = fmaf(fx_, e11, c6);
            const float dy0 = a10 - a00, dy1 = a11 - a01;
            const float b0 = fmaf(fy_, dy0, a00), b1 = fmaf(fy_, dy1, a01);
            const float dz = b1 - b0;
            W = fmaf(fz_, dz, b0);
            const float ex0 = fmaf(fy_, e10 - e00, e00), ex1 = fmaf(fy_, e11 - e01, e01);
            d0 = fmaf(fz_, ex1 - ex0, ex0);
            d1 = fmaf(fz_, dy1 - dy0, dy0);
            d2 = dz;
        }
        sm.dTs[R][0][P] = d0;
        sm.dTs[R][1][P] = d1;
        sm.dTs[R][2][P] = d2;
        (&sm.W[R][0][0])[P] = W;
        __syncthreads();

        // ------------------------------------------------------------- (B) q on plane k = p-1
        {
            const int k = p - 1;
            float qxv = 0.f, qyv = 0.f, qzv = 0.f;
            if (k >= z0 && k < z1) {  // CTA-uniform
                if (inter) {
                    const float* Wk = &sm.W[RB][0][0] + P;
                    const float wl = Wk[-1], wr = Wk[1], wu = Wk[-kE1X], wd = Wk[kE1X];
                    float gx = (wr - wl) * hx2;
                    float gy = (wd - wu) * hy2;
                    if (wface_b) {  // warp holds a position next to an x / y volume face
                        const float w0 = Wk[0];
                        if (fx) {
                            const float* cg = sm.colG[ex];
                            gx = fmaf(cg[0], wl, fmaf(cg[1], w0, cg[2] * wr));
                        }
                        if (fy) {
                            const float* rg = sm.rowG[ey];
                            gy = fmaf(rg[0], wu, fmaf(rg[1], w0, rg[2] * wd));
                        }
                    }
                    const int t = k - zb;
                    const float wzm = (&sm.W[RC][0][0])[P], wzp = (&sm.W[R][0][0])[P];
                    float gz;
                    if (sm.zi[t][2]) {  // z face plane (uniform): the exact one-sided rows
                        const float* zc = sm.zt[t];
                        gz = fmaf(zc[0], wzm, fmaf(zc[1], Wk[0], zc[2] * wzp));
                    } else {
                        gz = (wzp - wzm) * hz2;
                    }
                    // NGF ratio, distance term, q = dD/d grad W (ngf.py:70-112)
                    const float dot = fmaf(gx, rt.x, fmaf(gy, rt.y, gz * rt.z));
                    const float sq = fmaf(gx, gx, fmaf(gy, gy, fmaf(gz, gz, a.tau2)));
                    const float inv_nt = rsqrtf(sq);
                    const float r = fmaf(a.taurho, rt.w, dot) * inv_nt;
                    dacc += fmaf(-r, r, 1.0f);
                    const float t1 = r * inv_nt;
                    const float cf = a.neg_hbar * t1;
                    qxv = cf * fmaf(-t1, gx, rt.x);
                    qyv = cf * fmaf(-t1, gy, rt.y);
                    qzv = cf * fmaf(-t1, gz, rt.z);
                }
                // reference terms of plane p for the next step's (B)
                if (inter && p < z1) rt = __ldcs(a.RT + (size_t)p * ((size_t)a.nx * a.ny) + ij);
            }
            qz[RB] = qzv;
            (&sm.Qx[RB][0][1])[ey * (kE1X + 2) + ex] = qxv;
            (&sm.Qy[RB][1][0])[P] = qyv;
        }
        // staggered P^T passes of earlier completed deformation planes
        if (yz >= 0) {
            ypass(yz);
            yz = -1;
        }
        if (xz >= 0) {
            xpass();
            yz = xz;
            xz = -1;
        }

        // ------------------------------------------------------------- (C) j = p-2
        const int j = p - 2;
        if (j < jfirst || j > jlast) return;  // CTA-uniform
        const int t = j - zb;
        const float* qxj = &sm.Qx[RC][0][1] + ey * (kE1X + 2) + ex;
        const float* qyj = &sm.Qy[RC][1][0] + P;
        const float ql = qxj[-1], qr = qxj[1], qu = qyj[-kE1X], qd = qyj[kE1X];
        float sx = (ql - qr) * hx2;
        float sy = (qu - qd) * hy2;
        if (wface_c) {
            if (fx) {  // exact transposed face rows (warp.py:168-175)
                const float* ct = sm.colGt[ex];
                sx = fmaf(ct[0], ql, fmaf(ct[1], qxj[0], ct[2] * qr));
            }
            if (fy) {
                const float* rg = sm.rowGt[ey];
                sy = fmaf(rg[0], qu, fmaf(rg[1], qyj[0], rg[2] * qd));
            }
        }
        float sz;
        if (sm.zi[t][2]) {
            const float* zc = sm.zt[t];
            sz = fmaf(zc[3], qz[R], fmaf(zc[4], qz[RC], zc[5] * qz[RB]));
        } else {
            sz = (qz[R] - qz[RB]) * hz2;
        }
        const float sv = sx + sy + sz;
        const float w1 = sm.zt[t][6], w0 = sm.zt[t][7];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float g = sv * sm.dTs[RC][c][P];
            A0[c] = fmaf(w0, g, A0[c]);
            A1[c] = fmaf(w1, g, A1[c]);
        }
        // deformation plane i0z(j) is complete when the next image plane maps to the next
        // pair (the last plane of the chunk is flushed after the march)
        if (j < jlast && sm.zi[t][1] >= 1) {
            put_flush(A0);
            xz = sm.zi[t][0] - wzlo;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                A0[c] = A1[c];
                A1[c] = 0.f;
            }
        }
    }
};

template <int KX, int KY>
__global__ void __launch_bounds__(kNT, 2) k_march_lean(const __grid_constant__ FusedArgs<float> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    Lean<KX, KY> m(a, sm);
    const FusedPlan& fp = a.fp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- CTA geometry
    m.cta = blockIdx.x;
    const int tx = m.cta % fp.ntx, ty = (m.cta / fp.ntx) % fp.nty, tzc = m.cta / (fp.ntx * fp.nty);
    const int x0 = tx * 32, y0 = ty * kTYI;
    m.z0 = fp.zb_tab[tzc];
    m.z1 = fp.zb_tab[tzc + 1];
    m.zb = m.z0 - 1;
    m.jfirst = max(m.z0 - 1, 0);
    m.jlast = min(m.z1, a.nz - 1);
    m.wzlo = fp.win_z[tzc];

    // ---- this thread's position: row warps own columns 1..32 of one row, the last warp
    // the ring columns 0 and 33 of all rows
    if (warp < kE1Y) {
        m.ey = warp;
        m.ex = lane + 1;
    } else {
        m.ey = lane & 15;
        m.ex = lane < 16 ? 0 : kE1X - 1;
    }
    m.P = m.ey * kE1X + m.ex;
    m.x = x0 - 1 + m.ex;
    m.yy = y0 - 1 + m.ey;
    m.vol = m.x >= 0 && m.x < a.nx && m.yy >= 0 && m.yy < a.ny;
    m.inter = m.vol && warp >= 1 && warp <= kTYI;
    m.ij = m.vol ? (unsigned)(m.yy * a.nx + m.x) : 0u;
    {
        // a position needs the exact face coefficients where G or G^T differ from central
        const float hx2 = 0.5f * a.ihx, hy2 = 0.5f * a.ihy;
        float cm, c0, cp, gm, g0, gp;
        fd_coef<float>(m.x, a.nx, a.ihx, cm, c0, cp);
        fdt_coef<float>(m.x, a.nx, a.ihx, gm, g0, gp);
        m.fx = m.vol && !(cm == -hx2 && c0 == 0.f && cp == hx2 && gm == hx2 && g0 == 0.f && gp == -hx2);
        fd_coef<float>(m.yy, a.ny, a.ihy, cm, c0, cp);
        fdt_coef<float>(m.yy, a.ny, a.ihy, gm, g0, gp);
        m.fy = m.vol && !(cm == -hy2 && c0 == 0.f && cp == hy2 && gm == hy2 && g0 == 0.f && gp == -hy2);
    }
    m.wface_b = __any_sync(0xffffffffu, m.inter && (m.fx || m.fy));
    m.wface_c = __any_sync(0xffffffffu, m.fx || m.fy);

    // ---- shared tables
    for (int e = tid; e < kE1X; e += kNT) {
        const int i = x0 - 1 + e;
        fd_coef<float>(i, a.nx, a.ihx, sm.colG[e][0], sm.colG[e][1], sm.colG[e][2]);
        fdt_coef<float>(i, a.nx, a.ihx, sm.colGt[e][0], sm.colGt[e][1], sm.colGt[e][2]);
        const bool in = i >= 0 && i < a.nx;
        const int i0 = in ? a.i0x[i] : 0;
        sm.colP0[e] = i0;
        sm.colP1[e] = min(i0 + 1, a.ndx - 1);
        sm.colPw[e] = in ? a.w1x[i] : 0.f;
    }
    for (int e = tid; e < kE1Y; e += kNT) {
        const int jj = y0 - 1 + e;
        fd_coef<float>(jj, a.ny, a.ihy, sm.rowG[e][0], sm.rowG[e][1], sm.rowG[e][2]);
        fdt_coef<float>(jj, a.ny, a.ihy, sm.rowGt[e][0], sm.rowGt[e][1], sm.rowGt[e][2]);
        const bool in = jj >= 0 && jj < a.ny;
        const int i0 = in ? a.i0y[jj] : 0;
        sm.rowP0[e] = i0;
        sm.rowP1[e] = min(i0 + 1, a.ndy - 1);
        sm.rowPw[e] = in ? a.w1y[jj] : 0.f;
    }
    for (int t = tid; t < m.z1 + 2 - m.zb; t += kNT) {
        const int z = m.zb + t;
        float* zc = sm.zt[t];
        fd_coef<float>(z, a.nz, a.ihz, zc[0], zc[1], zc[2]);
        fdt_coef<float>(z, a.nz, a.ihz, zc[3], zc[4], zc[5]);
        const bool in = z >= 0 && z < a.nz;
        const float w1 = in ? a.w1z[z] : 0.f;
        zc[6] = w1;
        zc[7] = __fsub_rn(1.0f, w1);
        sm.zi[t][0] = in ? a.i0z[z] : 0;
        sm.zi[t][1] = (in && z + 1 < a.nz) ? a.i0z[z + 1] - a.i0z[z] : 2;
        const float hz2 = 0.5f * a.ihz;
        const bool central = zc[0] == -hz2 && zc[1] == 0.f && zc[2] == hz2 && zc[3] == hz2 && zc[4] == 0.f &&
                             zc[5] == -hz2;
        sm.zi[t][2] = central ? 0 : 1;
    }
    for (int t = tid; t < 3 * kE1Y * (kE1X + 2); t += kNT) (&sm.Qx[0][0][0])[t] = 0.f;
    for (int t = tid; t < 3 * (kE1Y + 2) * kE1X; t += kNT) (&sm.Qy[0][0][0])[t] = 0.f;
    {
        const int2* gx = reinterpret_cast<const int2*>(fp.lx) + (size_t)tx * fp.wx * KX;
        const int2* gy = reinterpret_cast<const int2*>(fp.ly) + (size_t)ty * fp.wy * KY;
        for (int t = tid; t < fp.wx * KX; t += kNT) sm.xl[t / KX][t % KX] = gx[t];
        for (int t = tid; t < fp.wy * KY; t += kNT) sm.yl[t / KY][t % KY] = gy[t];
    }
    // flush pass assignment: x pass (row, window column), y pass (window row, column)
    {
        unsigned xa = 0xffffu, ya = 0xffffu;
        if (tid < kE1Y * fp.wx) {
            const int r = tid / fp.wx;
            xa = (unsigned)r | (unsigned)(tid - r * fp.wx) << 8;
        }
        if (tid < fp.wy * fp.wx) {
            const int r = tid / fp.wx;
            ya = (unsigned)r | (unsigned)(tid - r * fp.wx) << 8;
        }
        m.fa = xa | ya << 16;
    }

    // ---- march state
    m.cur_zd = -1000;
    m.dacc = 0.f;
    m.xz = m.yz = -1;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        m.qz[r] = 0.f;
        m.ylo[r] = m.yhi[r] = m.A0[r] = m.A1[r] = 0.f;
    }
    m.rt = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    if (m.inter && m.z0 < m.z1) m.rt = __ldcs(a.RT + (size_t)m.z0 * ((size_t)a.nx * a.ny) + m.ij);

    // planes p = z0-1 .. z1+2: (A) on p, (B) on p-1, (C) on p-2
    const int pstart = m.z0 - 1;
    const int nsteps = (m.z1 + 2) - pstart + 1;
    for (int b = 0; b < nsteps; b += 3) {
        m.template step<0>(pstart + b);
        if (b + 1 < nsteps) m.template step<1>(pstart + b + 1);
        if (b + 2 < nsteps) m.template step<2>(pstart + b + 2);
    }

    // ---- drain the staggered passes, then the chunk's last deformation plane(s)
    __syncthreads();
    if (m.yz >= 0) m.ypass(m.yz);
    if (m.xz >= 0) {
        __syncthreads();
        m.xpass();
        __syncthreads();
        m.ypass(m.xz);
    }
    if (m.jfirst <= m.jlast) {
        const int zdl = sm.zi[m.jlast - m.zb][0];
        __syncthreads();
        m.put_flush(m.A0);
        __syncthreads();
        m.xpass();
        __syncthreads();
        m.ypass(zdl - m.wzlo);
        if (zdl + 1 <= a.ndz - 1) {
            m.put_flush(m.A1);  // Fb is free: every x pass reading it is behind a barrier
            __syncthreads();
            m.xpass();
            __syncthreads();
            m.ypass(zdl + 1 - m.wzlo);
        }
    }

    // ---- the CTA's D partial (fixed order: warp tree, then warps in order)
    double v = (double)m.dacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red[warp] = v;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kWarps; ++w) s += sm.red[w];
        a.dpart[blockIdx.x] = s;
    }
}

template <int KX, int KY>
static cudaError_t set_smem(size_t smem) {
    return cudaFuncSetAttribute(k_march_lean<KX, KY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace lean

size_t lean_smem(int, int) { return sizeof(lean::Smem); }

int lean_prepare(size_t smem) {
    static std::mutex mu;
    static size_t granted = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (smem <= granted) return 0;
    cudaError_t e = lean::set_smem<8, 8>(smem);
    if (e == cudaSuccess) e = lean::set_smem<4, 4>(smem);
    if (e == cudaSuccess) e = lean::set_smem<8, 4>(smem);
    if (e == cudaSuccess) e = lean::set_smem<4, 8>(smem);
    if (e == cudaSuccess) granted = smem;
    return (int)e;
}

void lean_launch(const FusedArgs<float>& a, cudaStream_t s) {
    const FusedPlan& fp = a.fp;
    if (fp.kx <= 4 && fp.ky <= 4)
        NGF_LAUNCH((lean::k_march_lean<4, 4>), fp.n_cta, lean::kNT, fp.smem_bytes, s, a);
    else if (fp.kx <= 4)
        NGF_LAUNCH((lean::k_march_lean<4, 8>), fp.n_cta, lean::kNT, fp.smem_bytes, s, a);
    else if (fp.ky <= 4)
        NGF_LAUNCH((lean::k_march_lean<8, 4>), fp.n_cta, lean::kNT, fp.smem_bytes, s, a);
    else
        NGF_LAUNCH((lean::k_march_lean<8, 8>), fp.n_cta, lean::kNT, fp.smem_bytes, s, a);
}

}  // namespace ngf
