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
// -- re-laid out so that a step costs about 0.7 of the classic march's instructions:
//   * one position per thread (no slot loops or per-slot flag decoding): 14 row warps,
//     2 ring-row warps and 1 ring-column warp cover the 34 x 16 tile + ring, and the tile
//     is 32 wide in x, so a 256-wide level is 8 tiles with no padding; 544 threads at 56
//     registers, two CTAs per SM;
//   * ONE __syncthreads per plane: W and the interpolant derivative live in 4-plane
//     shared rings aligned with the deformation cells, q_x and q_y in shared planes
//     double-buffered by parity; the z neighbours of q stay in registers;
//   * the trilinear value and derivative as f32x2 pairs (FFMA2) over the z corner pairs
//     (grid ratio 4);
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

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "fused_cfg.cuh"
#include "march_lean.cuh"

namespace ngf {
namespace lean {

// NGF_LEAN_CHECKS: trap on any shared-memory index outside its array (debug builds)
#ifdef NGF_LEAN_CHECKS
#define LEAN_CHECK(c) \
    do {              \
        if (!(c)) __trap(); \
    } while (0)
#else
#define LEAN_CHECK(c) \
    do {              \
    } while (0)
#endif

constexpr int kPlane = kE1Y * kE1X;  // positions, row stride 34 for every per-position plane
constexpr int kSink = kPlane;        // the position of ring-column lanes beyond 2 * kE1Y
constexpr int kPl = kPlane + kE1X + 2;  // per-position plane incl. the sink and its neighbours
constexpr int kFbPitch = kE1X + 1;   // Fb row pitch: 3 row + 16 column offset banks apart
constexpr int kWXP = kWXM + 1;       // Xr row pitch (odd)
static_assert(kE1Y * kFbPitch + 2 <= kPl, "Fb rows fit the per-position plane");
constexpr int kRing = 4;             // plane ring: slot = (plane - phase) mod 4, aligned with the
                                     // deformation cells at grid ratio 2 and 4 (steady blocks)

// events of a steady-state step (compile-time schedule, see Lean::block)
constexpr unsigned kEvA = 1, kEvF = 2, kEvX = 4, kEvY = 8, kEvA1 = 16;  // kEvA1: plane p+1 starts a cell
constexpr unsigned kEvXN = 32;  // plane p+2 starts a cell: stage its x-interpolated deformation rows

struct Smem {
    float W[kRing][kPl];                  // W of planes p-3 .. p (ring by (plane - phase) mod 4)
    float dT[kRing][3][kPl];              // interpolant derivative (times h), same ring
    float Qx[2][kPl + 2];                 // q_x at [P + 1] (ring columns, q = 0, pad the rows), by plane parity
    float Qy[2][kPl + 2 * kE1X];          // q_y at [P + 34]: one zero row each side
    float Fb[3][kPl];                     // completed deformation plane (z-reduced ghat / h), rows
                                          // of kFbPitch (bank-conflict-free x pass)
    float Xr[3][kE1Y][kWXP];           // x-reduced (odd pitch)
    float Xs[3][kWYM][kE1X];           // the next cell's deformation rows interpolated in x
    int2 xl[kKMax][kWXM];              // x pass: (E1 column, weight bits) per entry, window output
    int2 yl[kWYM][kKMax];              // y pass: (E1 row, weight bits)
    float colG[kE1X][3], colGt[kE1X][3], rowG[kE1Y][3], rowGt[kE1Y][3];
    int colP0[kE1X], colP1[kE1X], rowP0[kE1Y], rowP1[kE1Y];
    float colPw[kE1X], rowPw[kE1Y];
    unsigned fa[kNT];                  // flush pass assignment per thread
    double red[kWarps];
};

// TMA instances: the reference terms of the tile interior of a plane land here by one
// tensor copy per plane, issued two steps ahead into a 4-slot ring (slot = ring slot of the
// plane), one mbarrier per slot; appended to Smem (128-byte aligned) in their dynamic
// shared memory only
struct RtBuf {
    float4 v[kRing][kTYI][32];
    unsigned long long bar[kRing];
};
constexpr size_t kRtOff = (sizeof(Smem) + 127) / 128 * 128;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// the reference terms are read once: keep them out of L1 (room for the template lines;
// `profiles/r02_ab_rt_no_allocate.txt`: -0.3 % at 256^3, -0.6 % at 512^3 against ld.global.cs)
__device__ __forceinline__ float4 ld_rt_na(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ float lerp_x(float a0, float a1, float w, float w0) {
    // a0 * (1 - w) + a1 * w, each op correctly rounded (transfer.py:126)
    return __fadd_rn(__fmul_rn(a0, w0), __fmul_rn(a1, w));
}

// Per-level control in the kernel's parameter space (constant bank): indexed by the
// CTA-uniform plane counter, so every branch of the march is a uniform one.
constexpr unsigned kAdv = 1u << 16;    // i0z(z + 1) == i0z(z) + 1
constexpr int kFaceShift = 17;         // bits 17-19: z-face slot + 1 (0: central z rows)

// PACK (f32x2 trilinear) by default at grid ratio 4; the ratio-2 instances are at the
// register limit already (PACK spills there)
template <int RATIO, int K, int NXY = 0, bool PACK = (RATIO == 4), bool PIPE = false, bool TMA = false>
struct Lean {
    static constexpr int KX = K, KY = K;
    // NXY > 0: a square NXY x NXY image plane known at compile time, so the 8 template
    // corners of a position are one address plus immediate offsets and the plane stride of
    // the reference terms is a constant
    __device__ __forceinline__ unsigned nx_() const { return NXY ? (unsigned)NXY : (unsigned)a.nx; }
    __device__ __forceinline__ unsigned nxy_() const {
        return NXY ? (unsigned)NXY * (unsigned)NXY : (unsigned)a.nx * (unsigned)a.ny;
    }
    const FusedArgs<float>& a;
    const Ctl& c;
    Smem& sm;
    RtBuf* rb;  // TMA instances only
    int P;         // flat E1 index ey * 34 + ex of this thread's position
    unsigned ij;   // yy * nx + x (reference-term offset inside a plane)
    unsigned fl;   // bit 0: x face, bit 1: y face, bit 2: interior position
    float m_in;    // 1 for interior positions, else 0 (distance accumulation)
    bool bwarp;    // the warp holds interior positions (runs (B))
    bool wface_b, wface_c;
    int cta, z0, z1, pa0, pa1, jfirst, jlast, wzlo, pstart, pend;
    float ylo[3], yhi[3];
    float g[8], gfx, gfy, gfz;  // the template corners and cell fractions of the next (A2)
    float qz[kRing];
    bool xok;   // Xs holds the rows of the next cell (staged by a steady step two planes ago)
    float A0[3], A1[3];
    float4 rt;
    float dacc;

    __device__ __forceinline__ Lean(const FusedArgs<float>& a_, const Ctl& c_, Smem& sm_)
        : a(a_), c(c_), sm(sm_), rb(reinterpret_cast<RtBuf*>(reinterpret_cast<unsigned char*>(&sm_) + kRtOff)) {}

    // TMA: the tile interior's reference terms of plane q into ring slot `slot` (thread 0)
    __device__ __forceinline__ void issue_rt(int q, int slot) const {
        const unsigned b = smem_u32(&rb->bar[slot]), d = smem_u32(&rb->v[slot][0][0]);
        constexpr unsigned kBytes = sizeof(rb->v[0]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kBytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
            "[%6];" ::"r"(d),
            "l"(reinterpret_cast<uint64_t>(&c.rt_map)), "r"(0), "r"((int)blockIdx.x * 32), "r"((int)blockIdx.y * kTYI),
            "r"(q), "r"(b)
            : "memory");
    }
    // wait for plane k's terms in slot `slot` (the n-th fill of the slot in this chunk has
    // parity n & 1, n = (k - z0) / 4)
    __device__ __forceinline__ void wait_rt(int k, int slot) const {
        const unsigned b = smem_u32(&rb->bar[slot]), par = (unsigned)((k - z0) >> 2) & 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_RT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_RT_%=;\n}" ::"r"(b),
            "r"(par)
            : "memory");
    }

    __device__ __forceinline__ void load_yplane(int zd, float (&out)[3]) const {
        // P_xy y on def plane zd at this position's image (x, y): x then y (transfer.py:136-142)
        // (the sink lanes read a valid table entry; their samples are redirected to the pad)
        const int ey = min(P / kE1X, kE1Y - 1), ex = P - (P / kE1X) * kE1X;
        LEAN_CHECK(ex >= 0 && ex < kE1X && ey >= 0 && ey < kE1Y);
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

    // the x lerps of P_xy (transfer.py:136-142) for plane zd on the tile's deformation rows,
    // shared by all positions: one (row, column) per thread over the three components, on
    // the last warps (the ring-column and ring-row warps run no (B))
    __device__ __forceinline__ void stage_x(int zd) const {
        const int t = kNT - 1 - (int)threadIdx.x, wy = a.fp.wy;
        if (t < wy * kE1X) {
            const int r = t / kE1X, ex = t - r * kE1X;
            LEAN_CHECK(r >= 0 && r < kWYM && ex >= 0 && ex < kE1X);
            const int j = min(sm.rowP0[0] + r, a.ndy - 1);
            const int x0 = sm.colP0[ex], x1 = sm.colP1[ex];
            const float wx = sm.colPw[ex], wx0 = __fsub_rn(1.0f, wx);
            const unsigned mm = (unsigned)(a.ndx * a.ndy * a.ndz);
            const unsigned o = (unsigned)zd * (unsigned)(a.ndx * a.ndy) + (unsigned)(j * a.ndx);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const unsigned ok = o + (unsigned)k * mm;
                sm.Xs[k][r][ex] = lerp_x(__ldg(a.y + (ok + (unsigned)x0)), __ldg(a.y + (ok + (unsigned)x1)), wx, wx0);
            }
        }
    }

    // P_xy y of the staged plane at this position: the y lerp of two staged rows (the same
    // operations as load_yplane)
    __device__ __forceinline__ void yplane_from_x(float (&out)[3]) const {
        const int ey = min(P / kE1X, kE1Y - 1), ex = P - (P / kE1X) * kE1X;
        const int j0 = sm.rowP0[0], top = a.fp.wy - 1;
        // rows outside the volume carry index 0 in the tables (their samples go to the zero
        // pad whatever yhat is): clamp them onto staged rows, never read outside Xs
        const int r0 = min(max(sm.rowP0[ey] - j0, 0), top), r1 = min(max(sm.rowP1[ey] - j0, 0), top);
        LEAN_CHECK(ex >= 0 && ex < kE1X && ey >= 0 && ey < kE1Y && r0 >= 0 && r1 < kWYM && top < kWYM);
        const float wy = sm.rowPw[ey], wy0 = __fsub_rn(1.0f, wy);
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k] = lerp_x(sm.Xs[k][r0][ex], sm.Xs[k][r1][ex], wy, wy0);
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
    __device__ __forceinline__ void xpass() const {
        const unsigned f = sm.fa[threadIdx.x];
        const int xr_r = f & 0xff, xr_d = (f >> 8) & 0xff;
        LEAN_CHECK(xr_r == 0xff || (xr_r < kE1Y && xr_d < kWXM));
        if (xr_r != 0xff) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
            const float* fb = &sm.Fb[0][0] + xr_r * kFbPitch;
#pragma unroll
            for (int k = 0; k < KX; ++k) {
                const int2 e = sm.xl[k][xr_d];
                const float w = __int_as_float(e.y);
                LEAN_CHECK(e.x >= 0 && xr_r * kFbPitch + e.x < kPl);
                s0 = fmaf(w, fb[e.x], s0);
                s1 = fmaf(w, fb[kPl + e.x], s1);
                s2 = fmaf(w, fb[2 * kPl + e.x], s2);
            }
            sm.Xr[0][xr_r][xr_d] = s0;
            sm.Xr[1][xr_r][xr_d] = s1;
            sm.Xr[2][xr_r][xr_d] = s2;
        }
    }

    // y pass: Xr -> the CTA's window partial of deformation plane slot zs (1/h applied)
    __device__ __forceinline__ void ypass(int zs) const {
        const unsigned f = sm.fa[threadIdx.x];
        const int yp_dy = (f >> 16) & 0xff, yp_d = f >> 24;
        LEAN_CHECK(yp_dy == 0xff || (yp_dy < kWYM && yp_d < kWXM));
        if (yp_dy != 0xff) {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int k = 0; k < KY; ++k) {
                const int2 e = sm.yl[yp_dy][k];
                const float w = __int_as_float(e.y);
                LEAN_CHECK(e.x >= 0 && e.x < kE1Y);
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
        const int f = P + P / kE1X;  // row pitch kFbPitch (the sink lands past the last row)
        LEAN_CHECK(f >= 0 && f < kPl);
        sm.Fb[0][f] = acc[0];
        sm.Fb[1][f] = acc[1];
        sm.Fb[2][f] = acc[2];
    }

    __device__ __forceinline__ bool flushes(int j) const {
        // deformation plane i0z(j) is complete after (C) on plane j (the chunk's last one is
        // flushed after the march)
        return j >= jfirst && j < jlast && (c.zw[j] & kAdv);
    }

    // (A1) plane q: yhat = P y (the P_xy pair of the position in registers, shifted /
    // reloaded when q starts a deformation cell), the cell lookup and the 8 template corner
    // reads (outside the hull: the zero pad), left in g[] / f*; q outside the chunk's A
    // range gives zeros (W = 0, derivative 0)
    template <bool GEN, bool NEWCELL, int RS = 0>
    __device__ __forceinline__ void a1(int q) {
        if (GEN && (q < pa0 || q > pa1)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) g[k] = 0.f;
            gfx = gfy = gfz = 0.f;
            return;
        }
        const bool reload = GEN && q == pa0;
        if (reload || (GEN ? (c.zw[q - 1] & kAdv) != 0 : NEWCELL)) {
            const int zd = (int)(c.zw[q] & 0xffffu);
            if (reload) {
                load_yplane(zd, ylo);
            } else {
#pragma unroll
                for (int k = 0; k < 3; ++k) ylo[k] = yhi[k];
            }
            if (!GEN && !PIPE && xok)
                yplane_from_x(yhi);
            else
                load_yplane(min(zd + 1, a.ndz - 1), yhi);
        }
        const float wz = GEN ? c.w1[q] : c.w1pat[RS], wz0 = __fsub_rn(1.0f, wz);
        const float yh0 = __fadd_rn(__fmul_rn(ylo[0], wz0), __fmul_rn(yhi[0], wz));
        const float yh1 = __fadd_rn(__fmul_rn(ylo[1], wz0), __fmul_rn(yhi[1], wz));
        const float yh2 = __fadd_rn(__fmul_rn(ylo[2], wz0), __fmul_rn(yhi[2], wz));
        bool in = fl & 8u;  // position inside the volume (x / y)
        const int ix = cell(yh0, a.ox, a.ihx, a.nm1x, a.hix, in, gfx);
        const int iy = cell(yh1, a.oy, a.ihy, a.nm1y, a.hiy, in, gfy);
        const int iz = cell(yh2, a.oz, a.ihz, a.nm1z, a.hiz, in, gfz);
        const unsigned nx = nx_(), nxy = nxy_();
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
        if constexpr (NXY >= 512) {
            // large planes (little reuse of template lines across tiles): the rows the next
            // plane's corners will most likely read, one template plane up, into L1
            // (`profiles/r02_ab_l1_prefetch.txt`: 512^3 -2.9 %, 256^3 +1.8 %: large planes only)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(bz + nxy));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(byz + nxy));
        }
    }

    // (A2): the trilinear value and derivative (times h) from g[] / f* in lerp form
    // (warp.py:79-85, :111-120)
    __device__ __forceinline__ void a2(float& W, float& d0, float& d1, float& d2) const {
        if constexpr (PACK) {
            // the bottom / top z corner pairs as f32x2: one FFMA2 per pair of lerps
            const float2 m1 = make_float2(-1.f, -1.f);
            const float2 z0 = make_float2(g[0], g[4]), z1 = make_float2(g[1], g[5]);
            const float2 z2 = make_float2(g[2], g[6]), z3 = make_float2(g[3], g[7]);
            const float2 fx2 = make_float2(gfx, gfx), fy2 = make_float2(gfy, gfy);
            const float2 e0 = __ffma2_rn(z0, m1, z1), e1 = __ffma2_rn(z2, m1, z3);
            const float2 a0 = __ffma2_rn(fx2, e0, z0), a1v = __ffma2_rn(fx2, e1, z2);
            const float2 dy = __ffma2_rn(a0, m1, a1v);
            const float2 bb = __ffma2_rn(fy2, dy, a0);
            const float2 ex = __ffma2_rn(fy2, __ffma2_rn(e0, m1, e1), e0);
            const float dz = bb.y - bb.x;
            W = fmaf(gfz, dz, bb.x);
            d0 = fmaf(gfz, ex.y - ex.x, ex.x);
            d1 = fmaf(gfz, dy.y - dy.x, dy.x);
            d2 = dz;
        } else {
            const float e00 = g[1] - g[0], e10 = g[3] - g[2], e01 = g[5] - g[4], e11 = g[7] - g[6];
            const float a00 = fmaf(gfx, e00, g[0]), a10 = fmaf(gfx, e10, g[2]);
            const float a01 = fmaf(gfx, e01, g[4]), a11 = fmaf(gfx, e11, g[6]);
            const float dy0 = a10 - a00, dy1 = a11 - a01;
            const float b0 = fmaf(gfy, dy0, a00), b1 = fmaf(gfy, dy1, a01);
            const float dz = b1 - b0;
            W = fmaf(gfz, dz, b0);
            const float ex0 = fmaf(gfy, e10 - e00, e00), ex1 = fmaf(gfy, e11 - e01, e01);
            d0 = fmaf(gfz, ex1 - ex0, ex0);
            d1 = fmaf(gfz, dy1 - dy0, dy0);
            d2 = dz;
        }
    }

    // One plane step: (A) on p, (B) on p-1, (C) on p-2.  R = ring slot of plane p.  GEN: the
    // generic step (chunk edges, volume faces: every condition tested on the uniform plane
    // counter); otherwise a steady-state step whose events EV are known at compile time.
    template <int R, bool GEN, unsigned EV>
    __device__ __forceinline__ void step(int p) {
        constexpr int RB = (R + 3) & 3;  // plane p-1
        constexpr int RC = (R + 2) & 3;  // plane p-2
        constexpr int RD = (R + 1) & 3;  // plane p-3
        if (GEN && (p < pstart || p >= pend)) return;  // alignment padding of the loop

        // ------------------------------------------------------------- (A) plane p
        // PIPE: its gathers were issued by the previous step's (A1); else issue them now
        if constexpr (!PIPE) a1<GEN, (EV & kEvA) != 0, R>(p);
        float W, d0, d1, d2;
        a2(W, d0, d1, d2);
        sm.W[R][P] = W;
        sm.dT[R][0][P] = d0;
        sm.dT[R][1][P] = d1;
        sm.dT[R][2][P] = d2;
        __syncthreads();
        if constexpr (PIPE) a1<GEN, (EV & kEvA1) != 0, (R + 1) & 3>(p + 1);  // plane p+1's gathers in flight during (B), (C)
        // the x lerps of the cell starting at plane p+2 (read by its (A) after the next barrier;
        // the previous staging was read by (A) of plane p, before this barrier)
        if constexpr (!GEN && !PIPE && (EV & kEvXN) != 0) {
            stage_x(min((int)(c.zw[p + 2] & 0xffffu) + 1, a.ndz - 1));
            xok = true;
        }
        if constexpr (GEN) xok = false;
        // TMA: the reference terms of plane p+1 (used by (B) two steps later); its slot's
        // previous plane (p-3) was read by (B) of step p-2, before this barrier
        if constexpr (TMA) {
            if (threadIdx.x == 0 && (!GEN || (p + 1 >= z0 && p + 1 < z1))) issue_rt(p + 1, (R + 1) & 3);
        }

        // ------------------------------------------------------------- (B) q on plane k = p-1
        const int k = p - 1;
        if (!GEN || (k >= z0 && k < z1)) {
            if (bwarp) {
                if constexpr (TMA) {
                    wait_rt(k, RB);
                    rt = rb->v[RB][(threadIdx.x >> 5) - 1][threadIdx.x & 31];
                }
                const float* Wk = &sm.W[RB][P];
                const float wl = Wk[-1], wr = Wk[1], wu = Wk[-kE1X], wd = Wk[kE1X];
                const float wzm = sm.W[RC][P], wzp = sm.W[R][P];
                float gx, gy;
                if constexpr (PACK) {  // the x and y central differences as one f32x2 pair
                    const float2 gxy = __fmul2_rn(__fadd2_rn(make_float2(wr, wd), make_float2(-wl, -wu)),
                                                  make_float2(c.hx2, c.hy2));
                    gx = gxy.x;
                    gy = gxy.y;
                } else {
                    gx = (wr - wl) * c.hx2;
                    gy = (wd - wu) * c.hy2;
                }
                if (wface_b) {  // warp holds a position next to an x / y volume face
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
                if (GEN) {
                    const unsigned fz = c.zw[k] >> kFaceShift;
                    if (fz) {  // z face plane: the exact one-sided rows
                        const float* zc = c.faceG[fz - 1];
                        gz = fmaf(zc[0], wzm, fmaf(zc[1], Wk[0], zc[2] * wzp));
                    }
                }
                // NGF ratio, distance term, q = dD/d grad W (ngf.py:70-112); positions outside
                // the interior carry rt = 0, hence q = 0, and m_in = 0
                const float dot = fmaf(gx, rt.x, fmaf(gy, rt.y, gz * rt.z));
                const float sq = fmaf(gx, gx, fmaf(gy, gy, fmaf(gz, gz, a.tau2)));
                const float inv_nt = rsqrtf(sq);
                const float r = fmaf(a.taurho, rt.w, dot) * inv_nt;
                dacc = fmaf(m_in, fmaf(-r, r, 1.0f), dacc);
                const float t1 = r * inv_nt;
                const float cf = a.neg_hbar * t1;
                qz[RB] = cf * fmaf(-t1, gz, rt.z);
                if constexpr (PACK) {
                    const float2 qxy = __fmul2_rn(make_float2(cf, cf),
                                                  __ffma2_rn(make_float2(-t1, -t1), make_float2(gx, gy),
                                                             make_float2(rt.x, rt.y)));
                    sm.Qx[RB & 1][P + 1] = qxy.x;
                    sm.Qy[RB & 1][P + kE1X] = qxy.y;
                } else {
                    sm.Qx[RB & 1][P + 1] = cf * fmaf(-t1, gx, rt.x);
                    sm.Qy[RB & 1][P + kE1X] = cf * fmaf(-t1, gy, rt.y);
                }
                // reference terms of plane p for the next step's (B)
                if constexpr (!TMA)
                    if ((!GEN || p < z1) && (fl & 4u)) rt = ld_rt_na(a.RT + (size_t)p * nxy_() + ij);
            }
        } else if (GEN && bwarp) {  // no q on this plane (chunk edges)
            qz[RB] = 0.f;
            sm.Qx[RB & 1][P + 1] = 0.f;
            sm.Qy[RB & 1][P + kE1X] = 0.f;
        }
        // staggered P^T passes of the deformation planes completed two and one steps ago
        if (GEN ? flushes(p - 4) : (EV & kEvY) != 0) ypass((int)(c.zw[p - 4] & 0xffffu) - wzlo);
        if (GEN ? flushes(p - 3) : (EV & kEvX) != 0) xpass();

        // ------------------------------------------------------------- (C) j = p-2
        const int j = p - 2;
        if (GEN && (j < jfirst || j > jlast)) return;
        const float* qxj = &sm.Qx[RC & 1][P + 1];
        const float* qyj = &sm.Qy[RC & 1][P + kE1X];
        const float ql = qxj[-1], qr = qxj[1], qu = qyj[-kE1X], qd = qyj[kE1X];
        float sx, sy;
        if constexpr (PACK) {
            const float2 sxy = __fmul2_rn(__fadd2_rn(make_float2(ql, qu), make_float2(-qr, -qd)),
                                          make_float2(c.hx2, c.hy2));
            sx = sxy.x;
            sy = sxy.y;
        } else {
            sx = (ql - qr) * c.hx2;
            sy = (qu - qd) * c.hy2;
        }
        if (wface_c) {
            const int ey = P / kE1X, ex = P - ey * kE1X;
            if (fl & 1u) {  // exact transposed face rows (warp.py:168-175)
                const float* ct = sm.colGt[ex];
                sx = fmaf(ct[0], ql, fmaf(ct[1], qxj[0], ct[2] * qr));
            }
            if (fl & 2u) {
                const float* rg = sm.rowGt[ey];
                sy = fmaf(rg[0], qu, fmaf(rg[1], qyj[0], rg[2] * qd));
            }
        }
        float sz = (qz[RD] - qz[RB]) * c.hz2;
        if (GEN) {
            const unsigned fz = c.zw[j] >> kFaceShift;
            if (fz) {
                const float* zc = c.faceG[fz - 1];
                sz = fmaf(zc[3], qz[RD], fmaf(zc[4], qz[RC], zc[5] * qz[RB]));
            }
        }
        const float sv = sx + sy + sz;
        const float w1 = GEN ? c.w1[j] : c.w1pat[RC], w0 = __fsub_rn(1.0f, w1);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float g = sv * sm.dT[RC][q][P];
            if constexpr (PACK) {  // both deformation planes' accumulators in one FFMA2
                const float2 acc = __ffma2_rn(make_float2(w0, w1), make_float2(g, g), make_float2(A0[q], A1[q]));
                A0[q] = acc.x;
                A1[q] = acc.y;
            } else {
                A0[q] = fmaf(w0, g, A0[q]);
                A1[q] = fmaf(w1, g, A1[q]);
            }
        }
        if (GEN ? flushes(j) : (EV & kEvF) != 0) {
            put_flush(A0);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                A0[q] = A1[q];
                A1[q] = 0.f;
            }
        }
    }

    // four steps from plane p (p = phase mod 4)
    __device__ __forceinline__ void generic4(int p) {
        step<0, true, 0>(p);
        step<1, true, 0>(p + 1);
        step<2, true, 0>(p + 2);
        step<3, true, 0>(p + 3);
    }

    // four steady-state steps from a plane p that starts a deformation cell, away from the
    // chunk edges and the volume faces: the events follow the grid ratio (a new cell at
    // every RATIO-th plane, its predecessor flushed one step later, x and y passes one and
    // two steps after that)
    __device__ __forceinline__ void block(int p) {
        if constexpr (RATIO == 4) {
            step<0, false, kEvA>(p);
            step<1, false, kEvF>(p + 1);
            step<2, false, kEvX | kEvXN>(p + 2);
            step<3, false, kEvY | kEvA1>(p + 3);
        } else if constexpr (RATIO == 2) {
            step<0, false, kEvA | kEvX | kEvXN>(p);
            step<1, false, kEvF | kEvY | kEvA1>(p + 1);
            step<2, false, kEvA | kEvX | kEvXN>(p + 2);
            step<3, false, kEvF | kEvY | kEvA1>(p + 3);
        } else {
            generic4(p);
        }
    }
};

template <int RATIO, int K, int NXY, bool PACK = (RATIO == 4), bool PIPE = false, bool TMA = false>
__global__ void __launch_bounds__(kNT, 2) k_march_lean(const __grid_constant__ FusedArgs<float> a,
                                                       const __grid_constant__ Ctl c) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    Lean<RATIO, K, NXY, PACK, PIPE, TMA> m(a, c, sm);
    constexpr int KX = K, KY = K;
    const FusedPlan& fp = a.fp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- CTA geometry (uniform): grid (x tiles, y tiles, z chunks), dispatched chunk-major
    const int tx = blockIdx.x, ty = blockIdx.y, tzc = blockIdx.z + a.chunk0;
    m.cta = (tzc * fp.nty + ty) * fp.ntx + tx;
    const int x0 = tx * 32, y0 = ty * kTYI;
    m.z0 = c.zb[tzc];
    m.z1 = c.zb[tzc + 1];
    m.pa0 = max(m.z0 - 1, 0);
    m.pa1 = min(m.z1, a.nz - 1);
    m.jfirst = m.pa0;
    m.jlast = m.pa1;
    m.wzlo = c.wzlo[tzc];

    // ---- this thread's position: row warps own columns 1..32 of one row, the last warp
    // the ring columns 0 and 33 of all rows
    int ex, ey;
    bool has = true;  // ring-column lanes beyond 2 * kE1Y hold no position (the sink)
    if (warp < kE1Y) {
        ey = warp;
        ex = lane + 1;
    } else {
        has = lane < 2 * kE1Y;
        ey = has ? (lane < kE1Y ? lane : lane - kE1Y) : 0;
        ex = lane < kE1Y ? 0 : kE1X - 1;
    }
    m.P = has ? ey * kE1X + ex : kSink;
    const int x = x0 - 1 + ex, yy = y0 - 1 + ey;
    const bool vol = has && x >= 0 && x < a.nx && yy >= 0 && yy < a.ny;
    const bool inter = vol && warp >= 1 && warp <= kTYI;
    m.ij = vol ? (unsigned)(yy * a.nx + x) : 0u;
    bool fx, fy;
    {
        // a position needs the exact face coefficients where G or G^T differ from central
        const float hx2 = c.hx2, hy2 = c.hy2;
        float cm, c0, cp, gm, g0, gp;
        fd_coef<float>(x, a.nx, a.ihx, cm, c0, cp);
        fdt_coef<float>(x, a.nx, a.ihx, gm, g0, gp);
        fx = vol && !(cm == -hx2 && c0 == 0.f && cp == hx2 && gm == hx2 && g0 == 0.f && gp == -hx2);
        fd_coef<float>(yy, a.ny, a.ihy, cm, c0, cp);
        fdt_coef<float>(yy, a.ny, a.ihy, gm, g0, gp);
        fy = vol && !(cm == -hy2 && c0 == 0.f && cp == hy2 && gm == hy2 && g0 == 0.f && gp == -hy2);
    }
    m.fl = (fx ? 1u : 0u) | (fy ? 2u : 0u) | (inter ? 4u : 0u) | (vol ? 8u : 0u);
    m.m_in = inter ? 1.f : 0.f;
    m.bwarp = __any_sync(0xffffffffu, inter);
    m.wface_b = __any_sync(0xffffffffu, inter && (fx || fy));
    m.wface_c = __any_sync(0xffffffffu, fx || fy);

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
    for (int t = tid; t < 2 * (kPl + 2); t += kNT) (&sm.Qx[0][0])[t] = 0.f;
    for (int t = tid; t < 2 * (kPl + 2 * kE1X); t += kNT) (&sm.Qy[0][0])[t] = 0.f;
    {
        const int2* gx = reinterpret_cast<const int2*>(fp.lx) + (size_t)tx * fp.wx * KX;
        const int2* gy = reinterpret_cast<const int2*>(fp.ly) + (size_t)ty * fp.wy * KY;
        for (int t = tid; t < fp.wx * KX; t += kNT) sm.xl[t % KX][t / KX] = gx[t];
        for (int t = tid; t < fp.wy * KY; t += kNT) sm.yl[t / KY][t % KY] = gy[t];
        // flush pass assignment: x pass (row, window column), y pass (window row, column).
        // x pass: half-warps hold the 16 rows of one window column, the two halves of a
        // warp columns d and d + o whose image columns lie 16 banks apart (o = 16 / ratio):
        // with the Fb row pitch of 35 the reads of a warp are conflict-free and its entry
        // list reads are two broadcasts
        static_assert(kE1Y <= 16, "x pass: a half-warp per window column");
        unsigned xa = 0xffffu, ya = 0xffffu;
        {
            constexpr int o = RATIO == 2 ? 8 : 4;
            const int idx = 2 * warp + (lane >> 4);  // window column slot
            int d = idx;
            if ((idx / (2 * o) + 1) * (2 * o) <= fp.wx) {
                const int j = idx % (2 * o);
                d = (idx - j) + (j >> 1) + (j & 1) * o;
            }
            if (d < fp.wx && (lane & 15) < kE1Y) xa = (unsigned)(lane & 15) | (unsigned)d << 8;
        }
        if (tid < fp.wy * fp.wx) {
            const int r = tid / fp.wx;
            ya = (unsigned)r | (unsigned)(tid - r * fp.wx) << 8;
        }
        sm.fa[tid] = xa | ya << 16;
    }

    // ---- march state
    m.dacc = 0.f;
    m.xok = false;
#pragma unroll
    for (int r = 0; r < 3; ++r) m.ylo[r] = m.yhi[r] = m.A0[r] = m.A1[r] = 0.f;
#pragma unroll
    for (int r = 0; r < kRing; ++r) m.qz[r] = 0.f;
    m.rt = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (TMA) {
        if (tid == 0) {
            for (int r = 0; r < kRing; ++r)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&m.rb->bar[r])) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    __syncthreads();
    // launched as a programmatic dependent of the previous kernel in the stream: the
    // prologue above reads only the plan tables; y, the reference terms, the partials and
    // dpart wait for that kernel's completion here
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the post kernel (programmatic dependent launch) may be scheduled once every CTA of this
    // grid is here: its prologue (which reads y) then runs on the SMs the last wave leaves
    // idle, and it waits (griddepcontrol.wait) for this grid's completion before reading the
    // partials.  Not earlier: before this grid's own wait, the kernel that wrote y (this
    // grid's predecessor) may still be running.
    asm volatile("griddepcontrol.launch_dependents;");
    if constexpr (!TMA) {
        if (inter && m.z0 < m.z1) m.rt = ld_rt_na(a.RT + (size_t)m.z0 * ((size_t)a.nx * a.ny) + m.ij);
    }

    // planes p = z0-1 .. z1+2: (A) on p, (B) on p-1, (C) on p-2, in groups of four steps
    // aligned to the plane phase (ring slot = (p - phase) mod 4); groups inside the chunk's
    // steady range [s0, s1) run the compile-time event schedule
    m.pstart = m.z0 - 1;
    m.pend = m.z1 + 3;
    const int s0 = c.s0[tzc], s1 = c.s1[tzc];
    if constexpr (PIPE) m.template a1<true, false>(m.pstart);  // the first plane's gathers
    for (int p = m.pstart - ((m.pstart - c.phase) & 3); p < m.pend; p += 4) {
        if (p >= s0 && p + 4 <= s1)
            m.block(p);
        else
            m.generic4(p);
    }

    // ---- drain the staggered passes (planes completed in the last two steps), then the
    // chunk's last deformation plane(s)
    const int pend = m.pend;  // the first step not taken
    __syncthreads();
    if (m.flushes(pend - 4)) m.ypass((int)(c.zw[pend - 4] & 0xffffu) - m.wzlo);
    if (m.flushes(pend - 3)) {
        m.xpass();
        __syncthreads();
        m.ypass((int)(c.zw[pend - 3] & 0xffffu) - m.wzlo);
    }
    if (m.jfirst <= m.jlast) {
        const int zdl = (int)(c.zw[m.jlast] & 0xffffu);
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
        a.dpart[m.cta] = s;
    }
}

template <int RATIO, int K, int NXY, bool PACK = (RATIO == 4), bool PIPE = false, bool TMA = false>
static cudaError_t set_smem(size_t smem) {
    return cudaFuncSetAttribute(k_march_lean<RATIO, K, NXY, PACK, PIPE, TMA>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// square power-of-two image planes with a compile-time size (the pyramid levels of the
// configurations: 32 .. 512); any other plane runs the runtime-size instance.  The A/B
// instances (scalar trilinear, gathers across the barrier) exist for 128 and 256.
template <int RATIO, int K>
static cudaError_t set_smem_all(size_t smem) {
    cudaError_t e = set_smem<RATIO, K, 0>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 32>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 64>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 128>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 256>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 512>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 256, false>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 128, false>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 256, false, true>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 128, false, true>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 256, (RATIO == 4), false, true>(smem);
    if (e == cudaSuccess) e = set_smem<RATIO, K, 128, (RATIO == 4), false, true>(smem);
    return e;
}

static bool scalar_trilinear() {
    static const bool on = std::getenv("NGF_LEAN_PACK") && std::atoi(std::getenv("NGF_LEAN_PACK")) == 0;
    return on;
}
static bool piped() {
    static const bool on = std::getenv("NGF_LEAN_PIPE") && std::atoi(std::getenv("NGF_LEAN_PIPE")) != 0;
    return on;
}
static bool tma_rt() {
    static const bool on = std::getenv("NGF_LEAN_TMA") && std::atoi(std::getenv("NGF_LEAN_TMA")) != 0;
    return on;
}

template <int RATIO, int K>
static void launch_sized(const FusedArgs<float>& a, const Ctl& c, dim3 grid, size_t sb, cudaStream_t s) {
    const int n = a.nx == a.ny ? a.nx : 0;
    if (tma_rt() && c.rt_map_ok && n == 256) {
        launch_pdl(k_march_lean<RATIO, K, 256, (RATIO == 4), false, true>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    if (tma_rt() && c.rt_map_ok && n == 128) {
        launch_pdl(k_march_lean<RATIO, K, 128, (RATIO == 4), false, true>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    if (piped() && n == 256) {
        launch_pdl(k_march_lean<RATIO, K, 256, false, true>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    if (piped() && n == 128) {
        launch_pdl(k_march_lean<RATIO, K, 128, false, true>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    if (scalar_trilinear() && n == 256) {
        launch_pdl(k_march_lean<RATIO, K, 256, false>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    if (scalar_trilinear() && n == 128) {
        launch_pdl(k_march_lean<RATIO, K, 128, false>, grid, dim3(kNT), sb, s, a, c);
        return;
    }
    switch (n) {
        case 32: launch_pdl(k_march_lean<RATIO, K, 32>, grid, dim3(kNT), sb, s, a, c); break;
        case 64: launch_pdl(k_march_lean<RATIO, K, 64>, grid, dim3(kNT), sb, s, a, c); break;
        case 128: launch_pdl(k_march_lean<RATIO, K, 128>, grid, dim3(kNT), sb, s, a, c); break;
        case 256: launch_pdl(k_march_lean<RATIO, K, 256>, grid, dim3(kNT), sb, s, a, c); break;
        case 512: launch_pdl(k_march_lean<RATIO, K, 512>, grid, dim3(kNT), sb, s, a, c); break;
        default: launch_pdl(k_march_lean<RATIO, K, 0>, grid, dim3(kNT), sb, s, a, c); break;
    }
}

}  // namespace lean

size_t lean_smem(int, int) {
    return lean::tma_rt() ? lean::kRtOff + sizeof(lean::RtBuf) : sizeof(lean::Smem);
}

int lean_rt_map(lean::Ctl* c, const void* rt, int nx, int ny, int nz) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static const Encode encode = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return (Encode) nullptr;
        }
        return (Encode)f;
    }();
    c->rt_map_ok = 0;
    if (!encode || !rt) return 0;
    const cuuint64_t dims[4] = {4, (cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t strides[3] = {16, 16ull * nx, 16ull * nx * ny};
    const cuuint32_t box[4] = {4, 32, (cuuint32_t)lean::kTYI, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = encode(&c->rt_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(rt), dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    c->rt_map_ok = r == CUDA_SUCCESS ? 1 : 0;
    return 0;
}

int lean_prepare(size_t smem) {
    static std::mutex mu;
    static size_t granted = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (smem <= granted) return 0;
    cudaError_t e = lean::set_smem_all<4, 8>(smem);
    if (e == cudaSuccess) e = lean::set_smem_all<2, 4>(smem);
    if (e == cudaSuccess) e = lean::set_smem<2, 8, 0>(smem);
    if (e == cudaSuccess) e = lean::set_smem<0, 8, 0>(smem);
    if (e == cudaSuccess) granted = smem;
    return (int)e;
}

void lean_launch(const FusedArgs<float>& a, const lean::Ctl& c, cudaStream_t s) {
    const FusedPlan& fp = a.fp;
    const dim3 grid(fp.ntx, fp.nty, a.nchunks ? a.nchunks : fp.ntz);
    const int k = (fp.kx <= 4 && fp.ky <= 4) ? 4 : 8;
    if (c.ratio == 4 && k == 8)
        lean::launch_sized<4, 8>(a, c, grid, fp.smem_bytes, s);
    else if (c.ratio == 2 && k == 4)
        lean::launch_sized<2, 4>(a, c, grid, fp.smem_bytes, s);
    else if (c.ratio == 2)
        launch_pdl((lean::k_march_lean<2, 8, 0>), grid, dim3(lean::kNT), fp.smem_bytes, s, a, c);
    else
        launch_pdl((lean::k_march_lean<0, 8, 0>), grid, dim3(lean::kNT), fp.smem_bytes, s, a, c);
}

// The per-level control block (kernel parameters) from the host plan.
int lean_ctl_build(const int32_t* i0z, const float* w1z, int nz, int ndz, double hz, const std::vector<int>& bounds,
                   const std::vector<int>& wzlo, double hx, double hy, lean::Ctl* c) {
    using namespace lean;
    if (nz > kMaxZ || (int)bounds.size() - 1 > kMaxChunks || ndz > 0xffff) return NGF_EARG;
    std::memset(c, 0, sizeof(Ctl));
    c->nchunk = (int)bounds.size() - 1;
    for (size_t t = 0; t < bounds.size(); ++t) c->zb[t] = bounds[t];
    for (int t = 0; t < c->nchunk; ++t) c->wzlo[t] = wzlo[t];
    const float ihz = (float)(1.0 / hz);
    c->hx2 = 0.5f * (float)(1.0 / hx);
    c->hy2 = 0.5f * (float)(1.0 / hy);
    c->hz2 = 0.5f * ihz;
    const int faces[4] = {0, 1, nz - 2, nz - 1};
    for (int f = 0; f < 4; ++f) {
        fd_coef<float>(faces[f], nz, ihz, c->faceG[f][0], c->faceG[f][1], c->faceG[f][2]);
        fdt_coef<float>(faces[f], nz, ihz, c->faceG[f][3], c->faceG[f][4], c->faceG[f][5]);
    }
    for (int z = 0; z < nz; ++z) {
        unsigned w = (unsigned)i0z[z];
        if (z + 1 < nz && i0z[z + 1] == i0z[z] + 1) w |= kAdv;
        float cm, c0, cp, gm, g0, gp;
        fd_coef<float>(z, nz, ihz, cm, c0, cp);
        fdt_coef<float>(z, nz, ihz, gm, g0, gp);
        const bool central = cm == -c->hz2 && c0 == 0.f && cp == c->hz2 && gm == c->hz2 && g0 == 0.f &&
                             gp == -c->hz2;
        if (!central) {
            int slot = 0;
            for (int f = 0; f < 4; ++f)
                if (faces[f] == z) slot = f + 1;
            if (!slot) return NGF_EARG;  // a non-central row away from the faces cannot happen
            w |= (unsigned)slot << kFaceShift;
        }
        c->zw[z] = w;
        c->w1[z] = w1z[z];
    }
    // the steady-state schedule: find the cell period r in {4, 2} and the phase, then per
    // chunk the planes [s0, s1) whose four-step groups may run it; every plane there is
    // checked against the z map (a new cell exactly at p = phase mod r, no face rows)
    auto adv = [&](int z) { return z >= 0 && z + 1 < nz && i0z[z + 1] == i0z[z] + 1; };
    c->ratio = 0;
    c->phase = 0;
    for (int r : {4, 2}) {
        int first = -1;
        for (int z = 3; z + 1 < nz && first < 0; ++z)
            if (adv(z - 1)) first = z;  // a plane starting a cell, away from the low face
        if (first < 0) continue;
        int run = 0;  // planes after `first` that follow the period-r pattern
        for (int z = first; z < nz - 2; ++z) {
            if (adv(z - 1) != ((z - first) % r == 0)) break;
            ++run;
        }
        if (run >= 8) {
            c->ratio = r;
            c->phase = first & 3;
            break;
        }
    }
    if (c->ratio) {
        // the w1 pattern: four consecutive planes away from the faces, by (plane - phase) mod 4
        const int z0 = std::min(std::max(4, nz / 2), std::max(nz - 4, 0));
        for (int k = 0; k < 4 && z0 + k < nz; ++k) c->w1pat[((z0 + k - c->phase) % 4 + 4) % 4] = c->w1[z0 + k];
    }
    for (int t = 0; t < c->nchunk; ++t) {
        c->s0[t] = c->s1[t] = 0;
        if (!c->ratio) continue;
        const int z0 = bounds[t], z1 = bounds[t + 1];
        int lo = std::max(z0 + 2, 4);
        lo += ((c->phase - lo) % 4 + 4) % 4;  // first group start = phase (mod 4)
        const int hi = std::min(z1 - 1, nz - 2);  // last plane a steady step may be on
        // a group at s is valid when the z map follows the period on planes s-4 .. s+3 (the
        // passes of steps s .. s+3 refer back to flushes after planes s-4 .. s-1) and its (B)
        // / (C) planes use central z rows; the steady range is the first run of valid groups
        auto valid = [&](int s) {
            for (int p = s - 4; p <= s + 4; ++p) {
                const bool want = ((p - c->phase) % c->ratio + c->ratio) % c->ratio == 0;
                if (adv(p - 1) != want) return false;
            }
            // the steady steps take w1 of planes s-2 .. s+3 from the 4-plane pattern
            for (int p = s - 2; p <= s + 3; ++p)
                if (std::memcmp(&c->w1[p], &c->w1pat[((p - c->phase) % 4 + 4) % 4], sizeof(float)) != 0)
                    return false;
            for (int p = s; p < s + 4; ++p)
                if (c->zw[p - 1] >> kFaceShift || c->zw[p - 2] >> kFaceShift) return false;
            return true;
        };
        int s = lo;
        while (s + 3 <= hi && !valid(s)) s += 4;
        int e = s;
        while (e + 3 <= hi && valid(e)) e += 4;
        if (e > s) {
            c->s0[t] = s;
            c->s1[t] = e;
        }
    }
    return 0;
}

}  // namespace ngf
