// Fused objective/gradient evaluation (performance path), declarations.
#pragma once
#include "common.cuh"

namespace ngf {

// Tile geometry of the fused kernel: kTX x TY image voxels per CTA in x/y (TY per
// kernel variant), a ring of one voxel around it, marching cz planes in z.
constexpr int kTX = 32;
constexpr int kCzMax = 96;  // longest z chunk a CTA marches (shared z tables)

struct FusedPlan {
    // kernel variant (tile rows, threads per CTA, occupancy) and tiles
    int variant, ty, nthreads;
    int packed;  // two-slot float2 march (f32 variants with two slots per thread)
    int ntx, nty, ntz, cz;  // cz: largest z chunk
    int zlo, zhi;  // image planes evaluated (a z-slab for config-5 decomposition; 0, nz otherwise)
    // P^T windows: max sizes and per-tile lower def index (device arrays)
    int wx, wy, wz;
    const int32_t* win_x;  // [ntx]
    const int32_t* win_y;  // [nty]
    const int32_t* win_z;  // [ntz]
    const int32_t* zb_tab; // [ntz + 1] z chunk boundaries (image planes), chunk sizes non-increasing
    // reduce cover lists: per def index up to kCover (tile, offset) pairs, -1 terminated
    const int32_t* cov_x;  // [ndx * kCover * 2]
    const int32_t* cov_y;
    const int32_t* cov_z;
    // per-tile CSR of the transposed 1-D interpolation over the tile window (host-built):
    // x tile t: offsets [wx+1] then E1 column indices [2*(kTX+2)]; weights separately
    const int32_t* xcsr;  // [ntx][wx + 1 + 2*(kTX+2)]
    const int32_t* ycsr;  // [nty][wy + 1 + 2*(ty+2)]
    const void* xcw;      // [ntx][2*(kTX+2)] dtype weights
    const void* ycw;      // [nty][2*(ty+2)]
    int n_cta;
    size_t smem_bytes;
    // lean march (variant kLeanVariant, march_lean.cu): zero-pad offset after the template
    // (reads outside the image hull land there), entries per P^T window output, and the
    // per-tile (E1 column / row, weight bits) lists of the x and y passes
    unsigned pad_off;
    int kx, ky;
    const int32_t* lx;  // [ntx][wx][kx] int2
    const int32_t* ly;  // [nty][wy][ky] int2
    const void* lean_ctl;  // HOST pointer to the level's lean::Ctl (launch parameters)
};
constexpr int kLeanVariant = 6;
constexpr int kWsVariant = 7;
constexpr int kCover = 8;

struct LevelDev;  // defined in level.cu

}  // namespace ngf
