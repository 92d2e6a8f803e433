// Lean fused march (f32, sm_100a): declarations shared with the host planner (level.cu)
// and the dispatcher (eval_fused.cu).  See march_lean.cu for the design.
#pragma once
#include "fused_impl.cuh"

namespace ngf {
namespace lean {

// Tile: 32 x TYI interior image columns x rows, a one-voxel ring around it (34 x (TYI+2)
// positions).  Row warps 0..TYI+1 own the 32 columns x0..x0+31 of one E1 row each; one
// ring-column warp owns columns x0-1 and x0+32 of all TYI+2 rows (16 + 16 lanes), so
// every lane of every warp holds a position and the tile is exactly 32 wide in x.
constexpr int kTYI = 14;
constexpr int kE1X = 34, kE1Y = kTYI + 2;
constexpr int kWarps = kE1Y + 1;  // 17
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
struct Eligibility {
    bool ok;
    int kx, ky;  // entries per window output (4 or 8)
};

}  // namespace lean

int lean_prepare(size_t smem);
size_t lean_smem(int kx, int ky);
void lean_launch(const FusedArgs<float>& a, cudaStream_t s);

}  // namespace ngf
