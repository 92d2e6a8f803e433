// Fused objective/gradient evaluation (performance path), declarations.
#pragma once
#include "common.cuh"

namespace ngf {

// Tile geometry of the fused kernel: TX x TY image voxels per CTA in x/y, a ring
// of one voxel around it (E1 = (TX+2) x (TY+2)), marching CZ planes in z.
constexpr int kTX = 32;
constexpr int kTY = 20;
constexpr int kE1X = kTX + 2;              // 34
constexpr int kE1Y = kTY + 2;              // 22
constexpr int kE1 = kE1X * kE1Y;           // 748
constexpr int kThreads = 256;
constexpr int kSlots = (kE1 + kThreads - 1) / kThreads;  // 3
constexpr int kE2X = kTX + 4;              // padded q layout (36)
constexpr int kE2Y = kTY + 4;              // 24
constexpr int kE2 = kE2X * kE2Y;           // 864

struct FusedPlan {
    // tiles
    int ntx, nty, ntz, cz;
    // P^T windows: max sizes and per-tile lower def index (device arrays)
    int wx, wy, wz;
    const int32_t* win_x;  // [ntx]
    const int32_t* win_y;  // [nty]
    const int32_t* win_z;  // [ntz]
    // reduce cover lists: per def index up to kCover (tile, offset) pairs, -1 terminated
    const int32_t* cov_x;  // [ndx * kCover * 2]
    const int32_t* cov_y;
    const int32_t* cov_z;
    int n_cta;
    size_t smem_bytes;
};
constexpr int kCover = 8;

struct LevelDev;  // defined in level.cu

}  // namespace ngf
