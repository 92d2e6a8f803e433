// Lean fused march (f32, sm_100a): declarations shared with the host planner (level.cu)
// and the dispatcher (eval_fused.cu).  See march_lean.cu for the design.
#pragma once
#include <cuda.h>  // CUtensorMap (the encode entry point is fetched at run time)
#include <vector>

#include "fused_impl.cuh"

namespace ngf {
namespace lean {

// Tile: 32 x TYI interior image columns x rows, a one-voxel ring around it (34 x (TYI+2)
// positions).  Row warps 0..TYI+1 own the 32 columns x0..x0+31 of one E1 row each; one
// ring-column warp owns columns x0-1 (lanes 0..TYI+1) and x0+32 (lanes TYI+2..2 TYI+3) of
// all rows, its other lanes sink, and the tile is exactly 32 wide in x.  TYI 14: 544
// threads, two CTAs per SM at 56 registers (TYI 13: 512 threads at 64 registers, 2 % faster
// at 256^3, 5 % at 128^3, but a different f32 summation order of the gradient partials;
// kept at 14 so that the long registration runs stay comparable to the recorded ones).
#ifndef NGF_LEAN_TYI
#define NGF_LEAN_TYI 14
#endif
constexpr int kTYI = NGF_LEAN_TYI;
constexpr int kE1X = 34, kE1Y = kTYI + 2;
constexpr int kWarps = kE1Y + 1;  // the row warps + the ring-column warp
static_assert(2 * kE1Y <= 32, "the ring columns of all rows fit one warp");
constexpr int kNT = 32 * kWarps;  // 544
constexpr int kWXM = 20;          // max P^T window outputs in x (34 columns at grid ratio >= 2)
constexpr int kWYM = 12;          // max window outputs in y (16 rows at ratio >= 2)
constexpr int kKMax = 8;          // max image columns (rows) feeding one window output

// Host-side eligibility of a level for the lean march.  All of: f32, every axis of the
// image at least 4 voxels and the deformation grid at least 2 nodes, power-of-two image
// spacing (the cell lookup multiplies by the exact reciprocal), the z index map advancing
// by at most one node per image plane and never on two consecutive planes (every
// deformation plane spans >= 2 image planes: the staggered flush), window and entry
// counts within the compile-time bounds.
constexpr int kMaxZ = 1024;      // image planes
constexpr int kMaxChunks = 128;  // z chunks per level

// Per-level control of the march, passed as a kernel parameter (constant bank) and indexed
// by the CTA-uniform plane counter so that every branch of the march is uniform.
struct alignas(64) Ctl {
    CUtensorMap rt_map;       // TMA descriptor of the packed reference terms (4, nx, ny, nz) f32
    int rt_map_ok;            // rt_map was encoded (the TMA instances may run)
    int nchunk;
    int ratio;                // 2 or 4: deformation cells of `ratio` planes in the steady range; 0: none
    int phase;                // a deformation cell starts at every plane = phase (mod 4) in the steady range
    int s0[kMaxChunks];       // per chunk: steady four-step groups cover planes [s0, s1)
    int s1[kMaxChunks];
    int zb[kMaxChunks + 1];   // chunk boundaries (image planes)
    int wzlo[kMaxChunks];     // lowest deformation plane of each chunk's P^T window
    unsigned zw[kMaxZ];       // per image plane: i0z (bits 0-15), advance flag, z-face slot
    float w1[kMaxZ];          // f32(w1z)
    float w1pat[4];           // w1 of a plane in the steady ranges, by (plane - phase) mod 4:
                              // compile-time constant-bank operands there (no indexed load)
    float faceG[4][8];        // z = 0, 1, nz-2, nz-1: G (cm, c0, cp), G^T (gm, g0, gp)
    float hx2, hy2, hz2;      // 1 / (2 h): central differences
};

}  // namespace lean

int lean_prepare(size_t smem);
// warp-specialised march (march_ws.cu): same eligibility and control block, 32 x 13 tiles
constexpr int kWsTYI = 13, kWsNT = 1024;
size_t ws_smem();
int ws_prepare(size_t smem);
void ws_launch(const FusedArgs<float>& a, const lean::Ctl& c, cudaStream_t s);
size_t lean_smem(int kx, int ky);
void lean_launch(const FusedArgs<float>& a, const lean::Ctl& c, cudaStream_t s);
// the reference-term tensor map of a level (box: one tile interior of one plane); 0 or an error
int lean_rt_map(lean::Ctl* c, const void* rt, int nx, int ny, int nz);
int lean_ctl_build(const int32_t* i0z, const float* w1z, int nz, int ndz, double hz, const std::vector<int>& bounds,
                   const std::vector<int>& wzlo, double hx, double hy, lean::Ctl* c);

}  // namespace ngf
