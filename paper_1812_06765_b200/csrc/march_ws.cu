// Warp-specialised fused NGF objective/gradient march (f32, sm_100a).
//
// The pipeline of march_lean.cu -- (A) yhat, template gathers, W and the interpolant
// derivative (transfer.py:117-148, warp.py:64-127); (B) grad W, the NGF ratio, the distance
// term and q (warp.py:130-143, ngf.py:70-112); (C) G^T q times the derivative, z-first P^T
// (warp.py:159-184, transfer.py:151-192) -- split between two groups of warps of one
// 1024-thread CTA per SM:
//   * 16 PRODUCER warps run (A) plane after plane into a ring of kSlots shared-memory planes
//     (W and the derivative), each warp keeping the NEXT plane's 8 template gathers in flight
//     while it interpolates the current one (software pipelining: producers need few
//     registers);
//   * 16 CONSUMER warps run (B) on plane p-1 and (C) on plane p-2 with one consumer-only
//     named barrier per plane, and the staggered x / y P^T passes.
// The groups meet only at per-slot named barriers: FULL[s] (producers arrive after writing
// plane p into slot s, consumers wait before reading it) and FREE[s] (consumers arrive once
// they are done with a plane, producers wait before overwriting its slot).  There is no
// CTA-wide barrier per plane, so the gather latency of one plane overlaps the consumers'
// work on earlier planes and producers run up to kSlots - 2 planes ahead.
// Tile: 32 x 13 interior voxels + ring (34 x 15 = 510 positions); each group maps warp w
// to E1 row w (columns 1..32) for w < 15 and to the ring columns for w = 15.
// Determinism: fixed-order sums everywhere; no atomics.

#include <algorithm>
#include <cstring>
#include <mutex>

#include "fused_cfg.cuh"
#include "march_lean.cuh"

namespace ngf {
namespace ws {

constexpr int kTYI = 13, kE1X = 34, kE1Y = kTYI + 2;  // 15 rows
constexpr int kGroup = 16;                             // warps per group
constexpr int kNT = 2 * 32 * kGroup;                   // 1024
constexpr int kPlane = kE1Y * kE1X;                    // 510 positions
constexpr int kPl = kPlane + 2;                        // + sink (threads without a position) + pad
constexpr int kSink = kPlane;
constexpr int kSlots = 6;                              // W / derivative ring
constexpr int kQSlots = 4;                             // q ring (consumers may be one plane apart)
constexpr int kWXM = lean::kWXM, kWYM = lean::kWYM, kKMax = lean::kKMax;
// named barrier ids: 0 __syncthreads, 1 consumers, 2.. FULL[s], 2 + kSlots.. FREE[s]
constexpr int kBarCons = 1, kBarFull = 2, kBarFree = 2 + kSlots;
static_assert(kBarFree + kSlots <= 16, "named barriers");

struct Smem {
    float W[kSlots][kPl];
    float dT[kSlots][3][kPl];
    float Qx[kQSlots][kPl + 2];        // q_x at [P + 1]
    float Qy[kQSlots][kPl + 2 * kE1X]; // q_y at [P + 34]
    float Fb[3][kPl];
    float Xr[3][kE1Y][kWXM];
    int2 xl[kWXM][kKMax];
    int2 yl[kWYM][kKMax];
    float colG[kE1X][3], colGt[kE1X][3], rowG[kE1Y][3], rowGt[kE1Y][3];
    int colP0[kE1X], colP1[kE1X], rowP0[kE1Y], rowP1[kE1Y];
    float colPw[kE1X], rowPw[kE1Y];
    unsigned short xo[kE1Y * kWXM];    // x pass outputs: row | window column << 8
    unsigned short yo[kWYM * kWXM];    // y pass outputs
    double red[kGroup];
};

__device__ __forceinline__ void bar_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kNT) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kNT) : "memory"); }
__device__ __forceinline__ void bar_cons() {
    asm volatile("bar.sync %0, %1;" ::"r"(kBarCons), "r"(kNT / 2) : "memory");
}

__device__ __forceinline__ float lerp_x(float a0, float a1, float w, float w0) {
    // a0 * (1 - w) + a1 * w, each op correctly rounded (transfer.py:126)
    return __fadd_rn(__fmul_rn(a0, w0), __fmul_rn(a1, w));
}

constexpr unsigned kAdv = 1u << 16;
constexpr int kFaceShift = 17;

// position of a thread inside its group (row warps, then the ring-column warp)
struct Pos {
    int P, ex, ey, x, yy;
    bool has, vol;
};
__device__ __forceinline__ Pos position(int gw, int lane, int x0, int y0, int nx, int ny) {
    Pos q;
    if (gw < kE1Y) {
        q.ey = gw;
        q.ex = lane + 1;
        q.has = true;
    } else {
        q.has = lane < 2 * kE1Y;
        q.ey = q.has ? (lane < kE1Y ? lane : lane - kE1Y) : 0;
        q.ex = lane < kE1Y ? 0 : kE1X - 1;
    }
    q.P = q.has ? q.ey * kE1X + q.ex : kSink;
    q.x = x0 - 1 + q.ex;
    q.yy = y0 - 1 + q.ey;
    q.vol = q.has && q.x >= 0 && q.x < nx && q.yy >= 0 && q.yy < ny;
    return q;
}

struct Common {
    const FusedArgs<float>& a;
    const lean::Ctl& c;
    Smem& sm;
    int cta, z0, z1, pa0, pa1, jfirst, jlast, wzlo, pstart, pend;
    __device__ __forceinline__ Common(const FusedArgs<float>& a_, const lean::Ctl& c_, Smem& sm_)
        : a(a_), c(c_), sm(sm_) {}
    __device__ __forceinline__ int slot(int p) const { return (p - pstart) % kSlots; }
    __device__ __forceinline__ int qslot(int p) const { return (p - pstart) & (kQSlots - 1); }
};

// ------------------------------------------------------------------ producers: (A)
struct Producer : Common {
    int P;
    bool vol;
    int ex, ey;
    float ylo[3], yhi[3];
    __device__ __forceinline__ Producer(const FusedArgs<float>& a_, const lean::Ctl& c_, Smem& sm_) : Common(a_, c_, sm_) {}

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

    __device__ __forceinline__ int cell(float p, float o, float ih, float nm1, float hi, bool& in, float& f) const {
        const float t = __fmul_rn(__fsub_rn(p, o), ih);
        in = in && (__float_as_uint(t) <= __float_as_uint(nm1));  // NaN and t < 0 (incl. -0) fail
        const float fl = fminf(floorf(t), hi);
        f = t - fl;
        return (int)fl;
    }

    // gathers of plane q into g (zeros outside the A range)
    __device__ __forceinline__ void issue(int q, float (&g)[8], float& fx, float& fy, float& fz) {
        if (q < pa0 || q > pa1) {
#pragma unroll
            for (int k = 0; k < 8; ++k) g[k] = 0.f;
            fx = fy = fz = 0.f;
            return;
        }
        const int zd = (int)(c.zw[q] & 0xffffu);
        if (q == pa0) {
            load_yplane(zd, ylo);
            load_yplane(min(zd + 1, a.ndz - 1), yhi);
        } else if (c.zw[q - 1] & kAdv) {
#pragma unroll
            for (int k = 0; k < 3; ++k) ylo[k] = yhi[k];
            load_yplane(min(zd + 1, a.ndz - 1), yhi);
        }
        const float wz = c.w1[q], wz0 = __fsub_rn(1.0f, wz);
        const float yh0 = __fadd_rn(__fmul_rn(ylo[0], wz0), __fmul_rn(yhi[0], wz));
        const float yh1 = __fadd_rn(__fmul_rn(ylo[1], wz0), __fmul_rn(yhi[1], wz));
        const float yh2 = __fadd_rn(__fmul_rn(ylo[2], wz0), __fmul_rn(yhi[2], wz));
        bool in = vol;
        const int ix = cell(yh0, a.ox, a.ihx, a.nm1x, a.hix, in, fx);
        const int iy = cell(yh1, a.oy, a.ihy, a.nm1y, a.hiy, in, fy);
        const int iz = cell(yh2, a.oz, a.ihz, a.nm1z, a.hiz, in, fz);
        const unsigned nx = (unsigned)a.nx, nxy = nx * (unsigned)a.ny;
        const unsigned off = in ? (unsigned)iz * nxy + (unsigned)iy * nx + (unsigned)ix : a.fp.pad_off;
        const float* b = a.Tv + off;
        const float* by = b + nx;
        const float* bz = b + nxy;
        const float* byz = bz + nx;
        g[0] = __ldg(b);
        g[1] = __ldg(b + 1);
        g[2] = __ldg(by);
        g[3] = __ldg(by + 1);
        g[4] = __ldg(bz);
        g[5] = __ldg(bz + 1);
        g[6] = __ldg(byz);
        g[7] = __ldg(byz + 1);
    }

    __device__ __forceinline__ void store(int s, const float (&g)[8], float fx, float fy, float fz) {
        // trilinear value and derivative (times h) in lerp form (warp.py:79-85, :111-120)
        const float e00 = g[1] - g[0], e10 = g[3] - g[2], e01 = g[5] - g[4], e11 = g[7] - g[6];
        const float a00 = fmaf(fx, e00, g[0]), a10 = fmaf(fx, e10, g[2]);
        const float a01 = fmaf(fx, e01, g[4]), a11 = fmaf(fx, e11, g[6]);
        const float dy0 = a10 - a00, dy1 = a11 - a01;
        const float b0 = fmaf(fy, dy0, a00), b1 = fmaf(fy, dy1, a01);
        const float dz = b1 - b0;
        const float ex0 = fmaf(fy, e10 - e00, e00), ex1 = fmaf(fy, e11 - e01, e01);
        sm.W[s][P] = fmaf(fz, dz, b0);
        sm.dT[s][0][P] = fmaf(fz, ex1 - ex0, ex0);
        sm.dT[s][1][P] = fmaf(fz, dy1 - dy0, dy0);
        sm.dT[s][2][P] = dz;
    }

    // planes pstart .. pend-1, each into slot(q); the next plane's gathers in flight while
    // the current one is interpolated
    __device__ __forceinline__ void run() {
        float ga[8], gb[8], fa[3], fb[3];
        issue(pstart, ga, fa[0], fa[1], fa[2]);
        for (int q = pstart; q < pend; q += 2) {
            issue(q + 1, gb, fb[0], fb[1], fb[2]);  // beyond pend: zeros, never stored
            if (q - pstart >= kSlots) bar_sync(kBarFree + slot(q));
            store(slot(q), ga, fa[0], fa[1], fa[2]);
            bar_arrive(kBarFull + slot(q));
            if (q + 1 >= pend) break;
            issue(q + 2, ga, fa[0], fa[1], fa[2]);
            if (q + 1 - pstart >= kSlots) bar_sync(kBarFree + slot(q + 1));
            store(slot(q + 1), gb, fb[0], fb[1], fb[2]);
            bar_arrive(kBarFull + slot(q + 1));
        }
    }
};

// ------------------------------------------------------------------ consumers: (B), (C)
template <int K>
struct Consumer : Common {
    int P;
    unsigned ij;
    unsigned fl;  // bit 0: x face, bit 1: y face, bit 2: interior
    float m_in;
    bool bwarp, wface_b, wface_c;
    float qz[kQSlots];
    float A0[3], A1[3];
    float4 rt;
    float dacc;
    int gtid;  // thread index inside the group (P^T pass outputs)
    __device__ __forceinline__ Consumer(const FusedArgs<float>& a_, const lean::Ctl& c_, Smem& sm_) : Common(a_, c_, sm_) {}

    __device__ __forceinline__ bool flushes(int j) const { return j >= jfirst && j < jlast && (c.zw[j] & kAdv); }

    __device__ __forceinline__ void xpass() const {
        const int n = kE1Y * a.fp.wx;
        for (int o = gtid; o < n; o += kNT / 2) {
            const unsigned rd = sm.xo[o];
            const int xr_r = rd & 0xff, xr_d = rd >> 8;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
            const float* fb = &sm.Fb[0][0] + xr_r * kE1X;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int2 e = sm.xl[xr_d][k];
                const float w = __int_as_float(e.y);
                s0 = fmaf(w, fb[e.x], s0);
                s1 = fmaf(w, fb[kPl + e.x], s1);
                s2 = fmaf(w, fb[2 * kPl + e.x], s2);
            }
            sm.Xr[0][xr_r][xr_d] = s0;
            sm.Xr[1][xr_r][xr_d] = s1;
            sm.Xr[2][xr_r][xr_d] = s2;
        }
    }

    __device__ __forceinline__ void ypass(int zs) const {
        const int wx = a.fp.wx, wy = a.fp.wy, n = wy * wx;
        const size_t win = (size_t)a.fp.wz * wy * wx;
        for (int o = gtid; o < n; o += kNT / 2) {
            const unsigned rd = sm.yo[o];
            const int dyy = rd & 0xff, d = rd >> 8;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int2 e = sm.yl[dyy][k];
                const float w = __int_as_float(e.y);
                s0 = fmaf(w, sm.Xr[0][e.x][d], s0);
                s1 = fmaf(w, sm.Xr[1][e.x][d], s1);
                s2 = fmaf(w, sm.Xr[2][e.x][d], s2);
            }
            float* out = a.partial + (size_t)cta * 3 * win + (size_t)zs * wy * wx + dyy * wx + d;
            out[0] = s0 * a.ihx;
            out[win] = s1 * a.ihy;
            out[2 * win] = s2 * a.ihz;
        }
    }

    __device__ __forceinline__ void put_flush(const float (&acc)[3]) {
        sm.Fb[0][P] = acc[0];
        sm.Fb[1][P] = acc[1];
        sm.Fb[2][P] = acc[2];
    }

    // (B) on plane k (W of k-1, k, k+1 in slots), q into the q ring
    __device__ __forceinline__ void phaseB(int k) {
        const int qs = qslot(k);
        if (!(k >= z0 && k < z1)) {
            if (bwarp) {
#pragma unroll
                for (int i = 0; i < kQSlots; ++i)
                    if (i == qs) qz[i] = 0.f;
                sm.Qx[qs][P + 1] = 0.f;
                sm.Qy[qs][P + kE1X] = 0.f;
            }
            return;
        }
        if (!bwarp) return;
        const float* Wk = &sm.W[slot(k)][P];
        const float wl = Wk[-1], wr = Wk[1], wu = Wk[-kE1X], wd = Wk[kE1X];
        const float wzm = sm.W[slot(k - 1)][P], wzp = sm.W[slot(k + 1)][P];
        float gx = (wr - wl) * (0.5f * a.ihx);
        float gy = (wd - wu) * (0.5f * a.ihy);
        if (wface_b) {
            const int ey = P / kE1X, ex = P - ey * kE1X;
            const float w0 = Wk[0];
            if (fl & 1u) {
                const float* cg = sm.colG[ex];
                gx = fmaf(cg[0], wl, fmaf(cg[1], w0, cg[2] * wr));
            }
            if (fl & 2u) {
                const float* rg = sm.rowG[ey];
                gy = fmaf(rg[0], wu, fmaf(rg[1], w0, rg[2] * wd));
            }
        }
        float gz = (wzp - wzm) * c.hz2;
        const unsigned fz = c.zw[k] >> kFaceShift;
        if (fz) {
            const float* zc = c.faceG[fz - 1];
            gz = fmaf(zc[0], wzm, fmaf(zc[1], Wk[0], zc[2] * wzp));
        }
        const float dot = fmaf(gx, rt.x, fmaf(gy, rt.y, gz * rt.z));
        const float sq = fmaf(gx, gx, fmaf(gy, gy, fmaf(gz, gz, a.tau2)));
        const float inv_nt = rsqrtf(sq);
        const float r = fmaf(a.taurho, rt.w, dot) * inv_nt;
        dacc = fmaf(m_in, fmaf(-r, r, 1.0f), dacc);
        const float t1 = r * inv_nt;
        const float cf = a.neg_hbar * t1;
        const float qzv = cf * fmaf(-t1, gz, rt.z);
#pragma unroll
        for (int i = 0; i < kQSlots; ++i)
            if (i == qs) qz[i] = qzv;
        sm.Qx[qs][P + 1] = cf * fmaf(-t1, gx, rt.x);
        sm.Qy[qs][P + kE1X] = cf * fmaf(-t1, gy, rt.y);
        // reference terms of plane k+1 for the next (B)
        if (k + 1 < z1 && (fl & 4u)) rt = __ldcs(a.RT + (size_t)(k + 1) * ((size_t)a.nx * a.ny) + ij);
    }

    __device__ __forceinline__ float qz_at(int p) const {
        const int i = qslot(p);
        float v = qz[0];
#pragma unroll
        for (int k = 1; k < kQSlots; ++k)
            if (i == k) v = qz[k];
        return v;
    }

    // (C) on plane j
    __device__ __forceinline__ void phaseC(int j) {
        if (j < jfirst || j > jlast) return;
        const int qs = qslot(j);
        const float* qxj = &sm.Qx[qs][P + 1];
        const float* qyj = &sm.Qy[qs][P + kE1X];
        const float ql = qxj[-1], qr = qxj[1], qu = qyj[-kE1X], qd = qyj[kE1X];
        float sx = (ql - qr) * (0.5f * a.ihx);
        float sy = (qu - qd) * (0.5f * a.ihy);
        if (wface_c) {
            const int ey = P / kE1X, ex = P - ey * kE1X;
            if (fl & 1u) {
                const float* ct = sm.colGt[ex];
                sx = fmaf(ct[0], ql, fmaf(ct[1], qxj[0], ct[2] * qr));
            }
            if (fl & 2u) {
                const float* rg = sm.rowGt[ey];
                sy = fmaf(rg[0], qu, fmaf(rg[1], qyj[0], rg[2] * qd));
            }
        }
        const float qm = qz_at(j - 1), q0 = qz_at(j), qp = qz_at(j + 1);
        float sz = (qm - qp) * c.hz2;
        const unsigned fz = c.zw[j] >> kFaceShift;
        if (fz) {
            const float* zc = c.faceG[fz - 1];
            sz = fmaf(zc[3], qm, fmaf(zc[4], q0, zc[5] * qp));
        }
        const float sv = sx + sy + sz;
        const float w1 = c.w1[j], w0 = __fsub_rn(1.0f, w1);
        const int s = slot(j);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float gg = sv * sm.dT[s][q][P];
            A0[q] = fmaf(w0, gg, A0[q]);
            A1[q] = fmaf(w1, gg, A1[q]);
        }
        if (flushes(j)) {
            put_flush(A0);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                A0[q] = A1[q];
                A1[q] = 0.f;
            }
        }
    }

    // steps p = pstart .. pend-1: wait for plane p, (B) on p-1, consumer barrier, passes,
    // (C) on p-2, release plane p-2's slot
    __device__ __forceinline__ void run(int last_free) {
        for (int p = pstart; p < pend; ++p) {
            bar_sync(kBarFull + slot(p));
            phaseB(p - 1);
            bar_cons();
            if (flushes(p - 4)) ypass((int)(c.zw[p - 4] & 0xffffu) - wzlo);
            if (flushes(p - 3)) xpass();
            phaseC(p - 2);
            // plane p-2 is done (its W was last read by (B) on p-1, its derivative by (C))
            if (p - 2 >= pstart && p - 2 <= last_free) bar_arrive(kBarFree + slot(p - 2));
        }
    }
};

template <int K>
__global__ void __launch_bounds__(kNT, 1) k_march_ws(const __grid_constant__ FusedArgs<float> a,
                                                     const __grid_constant__ lean::Ctl c) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const FusedPlan& fp = a.fp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool producer = warp < kGroup;
    const int gw = producer ? warp : warp - kGroup;  // warp inside its group
    const int tx = blockIdx.x, ty = blockIdx.y, tzc = blockIdx.z;
    const int x0 = tx * 32, y0 = ty * kTYI;
    const int cta = (tzc * fp.nty + ty) * fp.ntx + tx;

    // ---- shared tables (all threads)
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
    for (int t = tid; t < kQSlots * (kPl + 2); t += kNT) (&sm.Qx[0][0])[t] = 0.f;
    for (int t = tid; t < kQSlots * (kPl + 2 * kE1X); t += kNT) (&sm.Qy[0][0])[t] = 0.f;
    {
        const int2* gx = reinterpret_cast<const int2*>(fp.lx) + (size_t)tx * fp.wx * K;
        const int2* gy = reinterpret_cast<const int2*>(fp.ly) + (size_t)ty * fp.wy * K;
        for (int t = tid; t < fp.wx * K; t += kNT) sm.xl[t / K][t % K] = gx[t];
        for (int t = tid; t < fp.wy * K; t += kNT) sm.yl[t / K][t % K] = gy[t];
        for (int t = tid; t < kE1Y * fp.wx; t += kNT) {
            const int r = t / fp.wx;
            sm.xo[t] = (unsigned short)(r | (t - r * fp.wx) << 8);
        }
        for (int t = tid; t < fp.wy * fp.wx; t += kNT) {
            const int r = t / fp.wx;
            sm.yo[t] = (unsigned short)(r | (t - r * fp.wx) << 8);
        }
    }
    __syncthreads();

    const Pos pos = position(gw, lane, x0, y0, a.nx, a.ny);
    const int z0 = c.zb[tzc], z1 = c.zb[tzc + 1];
    auto setup = [&](Common& m) {
        m.cta = cta;
        m.z0 = z0;
        m.z1 = z1;
        m.pa0 = max(z0 - 1, 0);
        m.pa1 = min(z1, a.nz - 1);
        m.jfirst = m.pa0;
        m.jlast = m.pa1;
        m.wzlo = c.wzlo[tzc];
        m.pstart = z0 - 1;
        m.pend = z1 + 3;
    };
    if (producer) {
        Producer m(a, c, sm);
        setup(m);
        m.P = pos.P;
        m.vol = pos.vol;
        m.ex = pos.ex;
        m.ey = pos.ey;
#pragma unroll
        for (int k = 0; k < 3; ++k) m.ylo[k] = m.yhi[k] = 0.f;
        m.run();
    } else {
        Consumer<K> m(a, c, sm);
        setup(m);
        m.P = pos.P;
        m.gtid = gw * 32 + lane;
        const bool inter = pos.vol && gw >= 1 && gw <= kTYI;
        m.ij = pos.vol ? (unsigned)(pos.yy * a.nx + pos.x) : 0u;
        bool fx, fy;
        {
            const float hx2 = 0.5f * a.ihx, hy2 = 0.5f * a.ihy;
            float cm, c0, cp, gm, g0, gp;
            fd_coef<float>(pos.x, a.nx, a.ihx, cm, c0, cp);
            fdt_coef<float>(pos.x, a.nx, a.ihx, gm, g0, gp);
            fx = pos.vol && !(cm == -hx2 && c0 == 0.f && cp == hx2 && gm == hx2 && g0 == 0.f && gp == -hx2);
            fd_coef<float>(pos.yy, a.ny, a.ihy, cm, c0, cp);
            fdt_coef<float>(pos.yy, a.ny, a.ihy, gm, g0, gp);
            fy = pos.vol && !(cm == -hy2 && c0 == 0.f && cp == hy2 && gm == hy2 && g0 == 0.f && gp == -hy2);
        }
        m.fl = (fx ? 1u : 0u) | (fy ? 2u : 0u) | (inter ? 4u : 0u);
        m.m_in = inter ? 1.f : 0.f;
        m.bwarp = __any_sync(0xffffffffu, inter);
        m.wface_b = __any_sync(0xffffffffu, inter && (fx || fy));
        m.wface_c = __any_sync(0xffffffffu, fx || fy);
        m.dacc = 0.f;
#pragma unroll
        for (int r = 0; r < 3; ++r) m.A0[r] = m.A1[r] = 0.f;
#pragma unroll
        for (int r = 0; r < kQSlots; ++r) m.qz[r] = 0.f;
        m.rt = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inter && z0 < z1) m.rt = __ldcs(a.RT + (size_t)z0 * ((size_t)a.nx * a.ny) + m.ij);
        // a FREE arrival only for the planes a producer will wait on (plane q + kSlots produced)
        m.run(m.pend - 1 - kSlots);

        // ---- drain the staggered passes, then the chunk's last deformation plane(s)
        const int pend = m.pend;
        bar_cons();
        if (m.flushes(pend - 4)) m.ypass((int)(c.zw[pend - 4] & 0xffffu) - m.wzlo);
        if (m.flushes(pend - 3)) {
            m.xpass();
            bar_cons();
            m.ypass((int)(c.zw[pend - 3] & 0xffffu) - m.wzlo);
        }
        if (m.jfirst <= m.jlast) {
            const int zdl = (int)(c.zw[m.jlast] & 0xffffu);
            bar_cons();
            m.put_flush(m.A0);
            bar_cons();
            m.xpass();
            bar_cons();
            m.ypass(zdl - m.wzlo);
            if (zdl + 1 <= a.ndz - 1) {
                m.put_flush(m.A1);
                bar_cons();
                m.xpass();
                bar_cons();
                m.ypass(zdl + 1 - m.wzlo);
            }
        }
        // ---- the CTA's D partial (fixed order: warp tree, then consumer warps in order)
        double v = (double)m.dacc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sm.red[gw] = v;
        bar_cons();
        if (gw == 0 && lane == 0) {
            double s = 0.0;
            for (int w = 0; w < kGroup; ++w) s += sm.red[w];
            a.dpart[cta] = s;
        }
    }
}

}  // namespace ws

size_t ws_smem() { return sizeof(ws::Smem); }

int ws_prepare(size_t smem) {
    static std::mutex mu;
    static size_t granted = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (smem <= granted) return 0;
    cudaError_t e = cudaFuncSetAttribute(ws::k_march_ws<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ws::k_march_ws<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) granted = smem;
    return (int)e;
}

void ws_launch(const FusedArgs<float>& a, const lean::Ctl& c, cudaStream_t s) {
    const FusedPlan& fp = a.fp;
    const dim3 grid(fp.ntx, fp.nty, fp.ntz);
    if (fp.kx <= 4 && fp.ky <= 4)
        NGF_LAUNCH((ws::k_march_ws<4>), grid, ws::kNT, fp.smem_bytes, s, a, c);
    else
        NGF_LAUNCH((ws::k_march_ws<8>), grid, ws::kNT, fp.smem_bytes, s, a, c);
}

}  // namespace ngf
