// Fused march: kernel-variant configurations and the compile-time shared-memory layout,
// shared by the march translation units (march_v*.cu) and the host dispatch (eval_fused.cu).
#pragma once
#include <type_traits>

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

// the opt-in two-slot float2 march (fused_pair.cuh) is built for the 32 x 12 / 256-thread
// shape only (it keeps the derivative ring in registers)
template <typename T, typename C>
constexpr bool kPaired = std::is_same<T, float>::value && C::S == 2 && !C::DTS && C::TY == 12 && C::NT == 256;

// per variant, compiled in march_v<n>.cu: set the kernels' dynamic shared-memory limit;
// launch the march for one evaluation
template <typename T, typename C> int march_prepare(size_t smem);
template <typename T, typename C> void march_launch(const FusedArgs<T>& a, cudaStream_t s);

}  // namespace ngf
