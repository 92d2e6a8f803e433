// Level objective: reference terms, fused/exact evaluation (objective.py:22-60).

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "eval_fused.cuh"
#include "fused_impl.cuh"
#include "march_lean.cuh"
#include "ops_exact.cuh"

namespace ngf {


struct LevelWork {
    void* yhat = nullptr;   // 3N
    void* W = nullptr;      // N
    void* terms = nullptr;  // N
    void* q = nullptr;      // 3N
    void* s = nullptr;      // N
    void* ghat = nullptr;   // 3N
    void* gD = nullptr;     // 3M
    void* cws = nullptr;    // 6M
    double* dws = nullptr;  // 8
};

// ngf_level_eval_host's pipelined form (lean march, page-locked host buffers): the z chunks
// are split into parts, each with its own stream; part i's march starts once its y planes
// are up, its post kernel finalises the deformation planes no later chunk touches and their
// gradient goes down while the later parts march.
constexpr int kPipeMax = 8;
struct PipeState {
    cudaStream_t st[kPipeMax] = {};
    cudaStream_t up = nullptr, down = nullptr;
    cudaEvent_t start = nullptr, fin = nullptr, evH[kPipeMax] = {}, evM[kPipeMax] = {}, evP[kPipeMax] = {};
};

}  // namespace ngf

struct ngf_level {
    int dtype;
    ngf_grid_t img, def;
    ngf_plan_t* plan;
    const void* T;
    void* Tpad;  // lean march: copy of T followed by a zero pad (reads outside the hull)
    ngf::lean::Ctl* ctl;  // lean march: per-level control block (kernel parameters)
    bool slab_terms;  // reference terms exist only on the z-slab (ngf_level_create_zslab)
    void* gR;   // 3N exact reference terms
    void* nR;   // N
    void* RT;   // packed N x 4
    double tau, rho, alpha;
    // fused plan
    ngf::FusedPlan fp;
    void* fp_blob;   // device: windows + covers
    void* partial;   // n_cta x 3 x wz x wy x wx
    double* dpart;   // n_cta
    double* spart;   // one (L u)^2 partial per k_post block
    int ns;          // capacity of spart (>= k_post blocks)
    int* flag;       // [0] non-finite y seen in this evaluation, [1] k_post block counter
    int timing;      // record events around the fused kernel
    int pt_variant;  // P^T variant of the exact path (0 gather, 1 scatter, 2 red-black)
    cudaEvent_t ev[2];
    ngf::LevelWork ex;
    // ngf_level_eval_host: device copies of x and the gradient, scalars (device, pinned)
    void* hx;
    void* hg;
    double* hsc;
    double* hsc_pin;
    cudaEvent_t done;  // completion of the last launch: destroy waits for it, not the device
    ngf::PipeState* pipe;  // ngf_level_eval_host's streams and events (created on first use)
    int pipe_req;          // parts of the pipelined host evaluation (0: default, 1: serial)
};

namespace ngf {

static bool is_pow2(double h) {
    int e;
    double m = std::frexp(h, &e);
    return m == 0.5;
}

static int tile_windows(const int32_t* i0, int n, int nd, int tile, int ring_lo, std::vector<int>& lo,
                        std::vector<int>& hi, int org = 0, int end = -1) {
    // tiles [org + t*tile, min(org + (t+1)*tile, end)) plus a one-voxel ring each side;
    // window = def indices touched = [i0(first ring voxel), i0(last ring voxel) + 1]
    if (end < 0) end = n;
    const int nt = (end - org + tile - 1) / tile;
    lo.resize(nt);
    hi.resize(nt);
    int wmax = 1;
    for (int t = 0; t < nt; ++t) {
        int a = org + t * tile - ring_lo;
        if (a < 0) a = 0;
        int b = std::min(org + t * tile + tile, end);  // ring voxel after the tile
        if (b > n - 1) b = n - 1;
        int l = i0[a];
        int h = nd > 1 ? i0[b] + 1 : 0;
        if (h > nd - 1) h = nd - 1;
        lo[t] = l;
        hi[t] = h;
        if (h - l + 1 > wmax) wmax = h - l + 1;
    }
    return wmax;
}

// windows of explicit z chunks [bounds[t], bounds[t+1]) plus a one-plane ring each side
static int chunk_windows(const int32_t* i0, int n, int nd, const std::vector<int>& bounds, std::vector<int>& lo,
                         std::vector<int>& hi) {
    const int nt = (int)bounds.size() - 1;
    lo.resize(nt);
    hi.resize(nt);
    int wmax = 1;
    for (int t = 0; t < nt; ++t) {
        const int a = std::max(bounds[t] - 1, 0);
        const int b = std::min(bounds[t + 1], n - 1);  // ring plane after the chunk
        const int l = i0[a];
        int h = nd > 1 ? i0[b] + 1 : 0;
        if (h > nd - 1) h = nd - 1;
        lo[t] = l;
        hi[t] = h;
        wmax = std::max(wmax, h - l + 1);
    }
    return wmax;
}

// Makespan of greedy list scheduling (the hardware CTA dispatcher in blockIdx order) of
// `classes` = (item count, item cost) in order on `slots` identical slots.
static double list_schedule(const std::vector<std::pair<int64_t, double>>& classes, int64_t slots) {
    std::map<double, int64_t> free_at{{0.0, slots}};
    double makespan = 0.0;
    for (const auto& cl : classes) {
        int64_t left = cl.first;
        while (left > 0) {
            auto it = free_at.begin();
            const double t = it->first;
            const int64_t k = std::min(left, it->second);
            it->second -= k;
            if (it->second == 0) free_at.erase(it);
            free_at[t + cl.second] += k;
            makespan = std::max(makespan, t + cl.second);
            left -= k;
        }
    }
    return makespan;
}

static bool build_cover(const std::vector<int>& lo, const std::vector<int>& hi, int nd,
                        std::vector<int32_t>& cov, int limit = kCover) {
    cov.assign((size_t)nd * kCover * 2, -1);
    for (int d = 0; d < nd; ++d) {
        int k = 0;
        for (int t = 0; t < (int)lo.size(); ++t) {
            if (d >= lo[t] && d <= hi[t]) {
                if (k >= limit) return false;
                cov[((size_t)d * kCover + k) * 2] = t;
                cov[((size_t)d * kCover + k) * 2 + 1] = d - lo[t];
                ++k;
            }
        }
    }
    return true;
}

// Can the lean march (march_lean.cu) evaluate this level?  f32, every image axis >= 4
// voxels and every deformation axis >= 2 nodes, power-of-two image spacing (exact
// reciprocal in the cell lookup), the z index map advancing by <= 1 node per image plane
// and never on two consecutive planes (the staggered P^T flush), and windows / entry counts
// within the kernel's compile-time bounds.  Returns the entries per window output (x, y).
static bool lean_eligible(const ngf_level* L, int* kx, int* ky, int tyi = lean::kTYI) {
    const ngf_plan_t* p = L->plan;
    if (L->dtype != NGF_F32 || std::getenv("NGF_NO_LEAN")) return false;
    for (int ax = 0; ax < 3; ++ax) {
        if (L->img.dims[ax] < 4 || L->def.dims[ax] < 2) return false;
        if (!is_pow2(L->img.spacing[ax])) return false;
    }
    const int nz = (int)L->img.dims[2];
    const int32_t* iz = p->h_i0[2];
    for (int z = 0; z + 1 < nz; ++z) {
        const int adv = iz[z + 1] - iz[z];
        if (adv < 0 || adv > 1) return false;
        if (adv == 1 && z + 2 < nz && iz[z + 2] - iz[z + 1] == 1) return false;
    }
    // entries per window output: image columns (rows) of a tile + ring feeding one node
    int k[2] = {0, 0};
    const int tile[2] = {kTX, tyi};
    for (int ax = 0; ax < 2; ++ax) {
        const int n = (int)L->img.dims[ax], nd = (int)L->def.dims[ax];
        const int32_t* i0 = p->h_i0[ax];
        for (int t = 0; t * tile[ax] < n; ++t) {
            std::map<int, int> cnt;
            for (int e = 0; e < tile[ax] + 2; ++e) {
                const int i = t * tile[ax] - 1 + e;
                if (i < 0 || i >= n) continue;
                // zero weights (clamped image columns before the first / after the last
                // node) contribute nothing and are left out of the lists
                const double w1 = p->h_w1[ax][i];
                if (1.0 - w1 != 0.0) ++cnt[i0[i]];
                if (nd > 1 && w1 != 0.0) ++cnt[i0[i] + 1];
            }
            for (auto& kv : cnt) k[ax] = std::max(k[ax], kv.second);
        }
    }
    if (k[0] > lean::kKMax || k[1] > lean::kKMax) return false;
    *kx = k[0] <= 4 ? 4 : 8;
    *ky = k[1] <= 4 ? 4 : 8;
    return true;
}

template <typename T>
static int fused_setup(ngf_level* L, int zlo, int zhi, cudaStream_t stream = 0) {
    const auto t_start = std::chrono::steady_clock::now();
    const ngf_plan_t* p = L->plan;
    const int nx = (int)L->img.dims[0], ny = (int)L->img.dims[1], nz = (int)L->img.dims[2];
    const int ndx = (int)L->def.dims[0], ndy = (int)L->def.dims[1], ndz = (int)L->def.dims[2];
    std::vector<int> xl, xh, yl, yh, zl, zh;
    FusedPlan& fp = L->fp;
    // Kernel variant and z chunking, chosen together by simulating the CTA dispatch:
    // every tile column is cut into nb chunks of B planes followed by the remainder in
    // m near-equal smaller chunks; CTAs are numbered chunk-major, so all columns' big
    // chunks are dispatched first and the small ones fill the last wave (longest
    // processing time first).  A chunk of c planes costs (c + 14) x plane cost: ~14 planes
    // of per-CTA fixed work (tables, ring planes, pipeline fill; fitted with
    // NGF_CHUNK_OVERHEAD sweeps at 256^3 .. 512^3), and a plane cost
    // relative to variant 1 (tools/sweep.py at 128^3 .. 512^3: 32 x 16 tiles of 320
    // threads with the derivative ring in shared memory take 1.16x the time of 32 x 12
    // tiles of 256 threads per plane for 1.33x the voxels).  Every
    // chunking must keep each def node covered by at most kCover chunks (k_post's sum).
    static const int kMinBlocks[] = {2, 2, 2, 2, 1, 1, 2, 1};
    static const double kPlaneCost[] = {1.6, 1.0, 1.16, 1.5, 1.0, 1.14, 1.0, 1.0};  // f64 (4, 5) relative to 4; lean / ws alone
    // the search depends only on the geometry (dims, slab, index maps), the dtype and the
    // tuning overrides: memoised per process, so repeated registrations of one size (a
    // batch of pairs, config 4) skip it (1.4 ms at 256^3, 4.9 ms at 512^3)
    int lean_kx = 8, lean_ky = 8;
    const char* fv = std::getenv("NGF_FUSED_VARIANT");
    const bool want_ws = fv && std::atoi(fv) % 8 == kWsVariant;
    const bool lean_ok = sizeof(T) == 4 && lean_eligible(L, &lean_kx, &lean_ky, want_ws ? kWsTYI : lean::kTYI);
    std::string key = lean_ok ? "lean:" : "classic:";
    {
        const char* ev[] = {"NGF_FUSED_VARIANT", "NGF_FUSED_CZ", "NGF_CHUNK_OVERHEAD"};
        key += std::to_string(sizeof(T)) + ":" + std::to_string(zlo) + ":" + std::to_string(zhi);
        for (const char* e : ev) key += std::string(":") + (std::getenv(e) ? std::getenv(e) : "-");
        const int nimg[3] = {nx, ny, nz}, ndef[3] = {ndx, ndy, ndz};
        for (int ax = 0; ax < 3; ++ax) {
            key += "|" + std::to_string(nimg[ax]) + "/" + std::to_string(ndef[ax]) + ":";
            uint64_t h = 1469598103934665603ull;  // FNV-1a of the axis index map
            for (int i = 0; i < nimg[ax]; ++i) h = (h ^ (uint32_t)p->h_i0[ax][i]) * 1099511628211ull;
            key += std::to_string(h);
        }
    }
    std::vector<int> bounds;
    int variant = -1;
    size_t n_choices = 0;
    static std::mutex plan_mu;
    static std::map<std::string, std::pair<int, std::vector<int>>> plan_cache;
    {
        std::lock_guard<std::mutex> lk(plan_mu);
        auto it = plan_cache.find(key);
        if (it != plan_cache.end()) {
            variant = it->second.first;
            bounds = it->second.second;
        }
    }
    if (variant < 0) {
        std::vector<int> cand;
        const char* env = std::getenv("NGF_FUSED_VARIANT");
        if (sizeof(T) == 8) {  // f64 shapes: 0, 4, 5
            const int v = env ? std::atoi(env) : -1;
            cand = (v == 0 || v == 4 || v == 5) ? std::vector<int>{v} : std::vector<int>{4, 5};
        } else if (env && ((std::atoi(env) % 8 != kLeanVariant && std::atoi(env) % 8 != kWsVariant) || lean_ok)) {
            const int v = std::atoi(env) % 8;  // f32 shapes: 0 .. 5, 6 = lean, 7 = warp-specialised
            cand = {v};
        } else if (lean_ok) {
            cand = {kLeanVariant};
        } else {
            cand = {1, 2};
        }
        const int nzs = zhi - zlo;
        const double ovh = std::getenv("NGF_CHUNK_OVERHEAD") ? std::atof(std::getenv("NGF_CHUNK_OVERHEAD")) : 14.0;
        const int forced_cz = std::getenv("NGF_FUSED_CZ") ? std::atoi(std::getenv("NGF_FUSED_CZ")) : 0;
        struct Choice {
            double cost;
            int variant;
            std::vector<int> sizes;
        };
        std::vector<Choice> choices;
        for (int v : cand) {
            int ty, nth;
            fused_variant_geom(v, &ty, &nth);
            std::vector<int> a, b;
            const int wx = tile_windows(p->h_i0[0], nx, ndx, kTX, 1, a, b);
            const int ntx = (int)a.size();
            const int wy = tile_windows(p->h_i0[1], ny, ndy, ty, 1, a, b);
            const int nty = (int)a.size();
            if (fused_smem<T>(v, wx, wy) > size_t(220) * 1024) continue;
            const int64_t cols = (int64_t)ntx * nty, slots = (int64_t)kSMs * kMinBlocks[v];
            auto add = [&](std::vector<int> sizes) {
                std::vector<std::pair<int64_t, double>> cls;
                for (int s : sizes) cls.push_back({cols, (s + ovh) * kPlaneCost[v]});
                choices.push_back({list_schedule(cls, slots), v, std::move(sizes)});
            };
            for (int B = std::min(nzs, kCzMax); B >= 1; --B) {
                if (forced_cz > 0 && B != std::min(forced_cz, nzs)) continue;
                // big-chunk counts that leave less than ~3 big chunks for the remainder
                for (int nb = std::max(1, nzs / B - 2); nb * B <= nzs; ++nb) {
                    const int r = nzs - nb * B;
                    std::vector<int> big(nb, B);
                    if (r == 0) {
                        add(big);
                        continue;
                    }
                    if (forced_cz > 0) {  // uniform chunks of the forced size
                        if (nb == nzs / B) {
                            big.push_back(r);
                            add(big);
                        }
                        continue;
                    }
                    for (int div = 1; div <= 4; ++div) {  // remainder in m chunks of <= B / div
                        const int cap = std::max(1, B / div);
                        const int m = (r + cap - 1) / cap;
                        std::vector<int> sizes = big;
                        for (int i = 0; i < m; ++i) sizes.push_back(r / m + (i < r % m ? 1 : 0));
                        std::sort(sizes.begin() + nb, sizes.end(), std::greater<int>());
                        add(sizes);
                    }
                }
            }
        }
        std::stable_sort(choices.begin(), choices.end(),
                         [](const Choice& x, const Choice& y) { return x.cost < y.cost; });
        // cheapest valid chunking; first among those whose def planes are covered by at most 4
        // chunks (k_post's unrolled partial sum -- more covers take its serial loop, which at
        // small sizes costs more than the march gains from the extra chunks)
        for (const int limit : {4, kCover}) {
            for (const Choice& ch : choices) {
                std::vector<int> bd(1, zlo), a, b;
                for (int s : ch.sizes) bd.push_back(bd.back() + s);
                chunk_windows(p->h_i0[2], nz, ndz, bd, a, b);
                std::vector<int32_t> cov;
                if (build_cover(a, b, ndz, cov, limit)) {
                    bounds = bd;
                    variant = ch.variant;
                    break;
                }
            }
            if (variant >= 0) break;
        }
        n_choices = choices.size();
        if (variant >= 0) {
            std::lock_guard<std::mutex> lk(plan_mu);
            plan_cache[key] = {variant, bounds};
        }
    }
    if (variant < 0) return NGF_EARG;
    const auto t_plan = std::chrono::steady_clock::now();
    fp.variant = variant;
    // two-slot float2 march: opt-in (measured 388 us vs 375 us for the scalar march at
    // 256^3 -- the FP issue slots it saves are spent on pair formation and masking)
    fp.packed = std::getenv("NGF_FUSED_PACKED") ? 1 : 0;
    fused_variant_geom(variant, &fp.ty, &fp.nthreads);
    fp.wx = tile_windows(p->h_i0[0], nx, ndx, kTX, 1, xl, xh);
    fp.wy = tile_windows(p->h_i0[1], ny, ndy, fp.ty, 1, yl, yh);
    fp.ntx = (int)xl.size();
    fp.nty = (int)yl.size();
    fp.smem_bytes = fused_smem<T>(variant, fp.wx, fp.wy);
    fp.cz = 0;
    for (size_t t = 0; t + 1 < bounds.size(); ++t) fp.cz = std::max(fp.cz, bounds[t + 1] - bounds[t]);
    fp.zlo = zlo;
    fp.zhi = zhi;
    fp.wz = chunk_windows(p->h_i0[2], nz, ndz, bounds, zl, zh);
    fp.ntz = (int)zl.size();
    fp.n_cta = fp.ntx * fp.nty * fp.ntz;
    std::vector<int32_t> cx, cy, cz_;
    if (!build_cover(xl, xh, ndx, cx) || !build_cover(yl, yh, ndy, cy) ||
        !build_cover(zl, zh, ndz, cz_))
        return NGF_EARG;
    // per-tile CSR of the transposed 1-D interpolation over the tile window
    // (transfer.py:82-101 restricted to the tile's columns incl. its ring)
    auto build_csr = [&](int axis, int tile, int ntile, int w, const std::vector<int>& lo,
                         std::vector<int32_t>& csr, std::vector<T>& wts) {
        const int ne = tile + 2, n = p->n_img[axis], nd = p->n_def[axis];
        const int stride = w + 1 + 2 * ne;
        csr.assign((size_t)ntile * stride, 0);
        wts.assign((size_t)ntile * 2 * ne, (T)0);
        for (int t = 0; t < ntile; ++t) {
            int32_t* off = csr.data() + (size_t)t * stride;
            int32_t* idx = off + w + 1;
            T* wt = wts.data() + (size_t)t * 2 * ne;
            int cnt = 0;
            for (int d = 0; d < w; ++d) {
                off[d] = cnt;
                for (int e = 0; e < ne; ++e) {
                    const int i = t * tile - 1 + e;
                    if (i < 0 || i >= n) continue;
                    const int dl = p->h_i0[axis][i] - lo[t];
                    const double w1 = p->h_w1[axis][i];
                    if (dl == d) {
                        idx[cnt] = e;
                        wt[cnt++] = (T)(1.0 - w1);
                    } else if (dl == d - 1 && nd > 1) {
                        idx[cnt] = e;
                        wt[cnt++] = (T)w1;
                    }
                }
            }
            off[w] = cnt;
        }
    };
    std::vector<int32_t> xcsr, ycsr;
    std::vector<T> xcw, ycw;
    build_csr(0, kTX, fp.ntx, fp.wx, xl, xcsr, xcw);
    build_csr(1, fp.ty, fp.nty, fp.wy, yl, ycsr, ycw);
    // lean march: per tile and window output, K (E1 index, f32 weight bits) entries in
    // ascending E1 order (the reference's gather order, transfer.py:89-96), zero-padded
    std::vector<int32_t> lxv(2), lyv(2);
    fp.kx = fp.ky = 0;
    auto build_list = [&](int axis, int tile, int ntile, int w, int K, const std::vector<int>& lo,
                          std::vector<int32_t>& out) {
        const int ne = tile + 2, n = p->n_img[axis], nd = p->n_def[axis];
        out.assign((size_t)ntile * w * K * 2, 0);
        for (int t = 0; t < ntile; ++t)
            for (int d = 0; d < w; ++d) {
                int32_t* ent = out.data() + ((size_t)t * w + d) * K * 2;
                int cnt = 0;
                for (int e = 0; e < ne; ++e) {
                    const int i = t * tile - 1 + e;
                    if (i < 0 || i >= n) continue;
                    const int dl = p->h_i0[axis][i] - lo[t];
                    const double w1 = p->h_w1[axis][i];
                    float wt;
                    if (dl == d) wt = (float)(1.0 - w1);
                    else if (dl == d - 1 && nd > 1) wt = (float)w1;
                    else continue;
                    if (wt == 0.0f && (dl == d ? 1.0 - w1 : w1) == 0.0) continue;  // exact zero weight
                    if (cnt < K) {
                        ent[2 * cnt] = e;
                        std::memcpy(&ent[2 * cnt + 1], &wt, 4);
                    }
                    ++cnt;
                }
            }
    };
    if (variant == kLeanVariant || variant == kWsVariant) {
        fp.kx = lean_kx;
        fp.ky = lean_ky;
        if (!L->ctl) L->ctl = new lean::Ctl();
        std::vector<float> w1z(nz);
        for (int z = 0; z < nz; ++z) w1z[z] = (float)p->h_w1[2][z];
        std::vector<int> wz(zl.begin(), zl.end());
        if (int rc = lean_ctl_build(p->h_i0[2], w1z.data(), nz, ndz, L->img.spacing[2], bounds, wz,
                                    L->img.spacing[0], L->img.spacing[1], L->ctl))
            return rc;
        lean_rt_map(L->ctl, L->RT, nx, ny, nz);
        fp.lean_ctl = L->ctl;
        build_list(0, kTX, fp.ntx, fp.wx, fp.kx, xl, lxv);
        build_list(1, fp.ty, fp.nty, fp.wy, fp.ky, yl, lyv);
        const size_t n = (size_t)nx * ny * nz;
        fp.pad_off = (unsigned)n;
        if (!L->Tpad) {
            const size_t pad = (size_t)nx * ny + nx + 64;
            NGF_CUDA((cudaError_t)dev_alloc(&L->Tpad, (n + pad) * sizeof(float)));
            NGF_CUDA(cudaStreamSynchronize(0));  // the pool allocation (stream 0) before use on `stream`
            NGF_CUDA(cudaMemcpyAsync(L->Tpad, L->T, n * sizeof(float), cudaMemcpyDeviceToDevice, stream));
            NGF_CUDA(cudaMemsetAsync((float*)L->Tpad + n, 0, pad * sizeof(float), stream));
        }
    }
    std::vector<int32_t> blob;
    auto app = [&](const void* v, size_t bytes) {
        size_t off = blob.size();
        blob.resize(off + (bytes + 3) / 4);
        std::memcpy(blob.data() + off, v, bytes);
        while (blob.size() % 64) blob.push_back(0);
        return off;
    };
    std::vector<int32_t> wxv(xl.begin(), xl.end()), wyv(yl.begin(), yl.end()), wzv(zl.begin(), zl.end());
    std::vector<int32_t> zbv(bounds.begin(), bounds.end());
    auto appv = [&](const std::vector<int32_t>& v) { return app(v.data(), v.size() * 4); };
    size_t o_wx = appv(wxv), o_wy = appv(wyv), o_wz = appv(wzv), o_cx = appv(cx), o_cy = appv(cy),
           o_cz = appv(cz_), o_zb = appv(zbv), o_xcsr = appv(xcsr), o_ycsr = appv(ycsr),
           o_xcw = app(xcw.data(), xcw.size() * sizeof(T)), o_ycw = app(ycw.data(), ycw.size() * sizeof(T)),
           o_lx = appv(lxv), o_ly = appv(lyv);
    NGF_CUDA((cudaError_t)dev_alloc((void**)&L->fp_blob, blob.size() * 4));
    NGF_CUDA((cudaError_t)upload_blocking(L->fp_blob, blob.data(), blob.size() * 4));
    const int32_t* b = (const int32_t*)L->fp_blob;
    fp.win_x = b + o_wx;
    fp.win_y = b + o_wy;
    fp.win_z = b + o_wz;
    fp.cov_x = b + o_cx;
    fp.cov_y = b + o_cy;
    fp.cov_z = b + o_cz;
    fp.zb_tab = b + o_zb;
    fp.xcsr = b + o_xcsr;
    fp.ycsr = b + o_ycsr;
    fp.xcw = b + o_xcw;
    fp.ycw = b + o_ycw;
    fp.lx = b + o_lx;
    fp.ly = b + o_ly;
    const size_t win = (size_t)fp.wz * fp.wy * fp.wx;
    NGF_CUDA((cudaError_t)dev_alloc((void**)&L->partial, (size_t)fp.n_cta * 3 * win * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&L->dpart, (size_t)fp.n_cta * sizeof(double)));
    L->ns = (int)(((L->def.dims[0] + 31) / 32) * ((L->def.dims[1] + 7) / 8) * 3 * L->def.dims[2]);
    NGF_CUDA((cudaError_t)dev_alloc((void**)&L->spart, (size_t)L->ns * sizeof(double)));
    if (std::getenv("NGF_SETUP_DEBUG")) {
        const auto t_end = std::chrono::steady_clock::now();
        std::fprintf(stderr, "fused_setup %dx%dx%d: plan search %.3f ms (%zu choices; 0 = cached), tables+upload %.3f ms\n",
                     nx, ny, nz, std::chrono::duration<double, std::milli>(t_plan - t_start).count(),
                     n_choices, std::chrono::duration<double, std::milli>(t_end - t_plan).count());
    }
    return fused_prepare<T>(variant, fp.smem_bytes);
}

template <typename T>
static FusedArgs<T> fused_args(const ngf_level* L, const void* y) {
    FusedArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.nx = (int)L->img.dims[0];
    a.ny = (int)L->img.dims[1];
    a.nz = (int)L->img.dims[2];
    a.ndx = (int)L->def.dims[0];
    a.ndy = (int)L->def.dims[1];
    a.ndz = (int)L->def.dims[2];
    a.ox = (T)L->img.origin[0];
    a.oy = (T)L->img.origin[1];
    a.oz = (T)L->img.origin[2];
    a.hx = (T)L->img.spacing[0];
    a.hy = (T)L->img.spacing[1];
    a.hz = (T)L->img.spacing[2];
    a.ihx = (T)1 / a.hx;
    a.ihy = (T)1 / a.hy;
    a.ihz = (T)1 / a.hz;
    a.pow2x = is_pow2((double)a.hx);
    a.pow2y = is_pow2((double)a.hy);
    a.pow2z = is_pow2((double)a.hz);
    const ngf_plan_t* p = L->plan;
    a.i0x = p->axes[0].i0;
    a.i0y = p->axes[1].i0;
    a.i0z = p->axes[2].i0;
    a.w1x = w1_host_sel<T>(p->axes[0]);
    a.w1y = w1_host_sel<T>(p->axes[1]);
    a.w1z = w1_host_sel<T>(p->axes[2]);
    a.nm1x = (T)(a.nx - 1);
    a.nm1y = (T)(a.ny - 1);
    a.nm1z = (T)(a.nz - 1);
    a.hix = (T)(a.nx > 2 ? a.nx - 2 : 0);
    a.hiy = (T)(a.ny > 2 ? a.ny - 2 : 0);
    a.hiz = (T)(a.nz > 2 ? a.nz - 2 : 0);
    a.Tv = (const T*)(L->fp.variant == kLeanVariant || L->fp.variant == kWsVariant ? L->Tpad : L->T);
    a.RT = (const V4T<T>*)L->RT;
    a.y = (const T*)y;
    a.partial = (T*)L->partial;
    a.dpart = L->dpart;
    const T tau = (T)L->tau;
    a.tau2 = tau * tau;
    a.taurho = (T)(L->tau * L->rho);
    const double hbar = L->img.spacing[0] * L->img.spacing[1] * L->img.spacing[2];
    a.neg_hbar = (T)(-hbar);
    a.half_hbar = hbar / 2;
    a.fp = L->fp;
    return a;
}

template <typename T>
static int exact_alloc(ngf_level* L) {
    LevelWork& w = L->ex;
    if (w.yhat) return 0;
    const int64_t n = grid_n(L->img), m = grid_n(L->def);
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.yhat, 3 * n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.W, n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.terms, n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.q, 3 * n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.s, n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.ghat, 3 * n * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.gD, 3 * m * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.cws, 6 * m * sizeof(T)));
    NGF_CUDA((cudaError_t)dev_alloc((void**)&w.dws, 8 * sizeof(double)));
    return 0;
}

template <typename T>
__global__ void k_nonfinite(const T* __restrict__ y, int64_t n, int* flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(y[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static int fused_part(ngf_level* L, const void* y, void* grad, double* scal, cudaStream_t s, int part) {
    cudaEvent_t e0 = L->timing ? L->ev[0] : nullptr, e1 = L->timing ? L->ev[1] : nullptr;
    if (L->dtype == NGF_F32) {
        FusedArgs<float> a = fused_args<float>(L, y);
        return fused_eval_launch<float>(a, L->def, L->alpha, L->spart, L->ns, L->flag,
                                        (float*)grad, scal, s, e0, e1, part);
    }
    FusedArgs<double> a = fused_args<double>(L, y);
    return fused_eval_launch<double>(a, L->def, L->alpha, L->spart, L->ns, L->flag,
                                     (double*)grad, scal, s, e0, e1, part);
}

__global__ void k_finish_exact(const double* D, const double* S, double alpha, int* flag, double* out) {
    // J = D + alpha * S in python floats (objective.py:50-52); a non-finite trial point
    // gives J = inf to force a backtrack (objective.py:55-57)
    out[0] = *flag ? INFINITY : *D + alpha * *S;
    *flag = 0;
    out[1] = *D;
    out[2] = *S;
}

template <typename T>
static int eval_exact(ngf_level* L, const void* y, void* grad, double* scal, cudaStream_t s) {
    int rc = exact_alloc<T>(L);
    if (rc) return rc;
    LevelWork& w = L->ex;
    const int64_t n = grid_n(L->img);
    const double hbar = L->img.spacing[0] * L->img.spacing[1] * L->img.spacing[2];
    if ((rc = apply_P_impl<T>(L->plan, (const T*)y, (T*)w.yhat, s))) return rc;
    if ((rc = warp_impl<T>(&L->img, (const T*)L->T, (const T*)w.yhat, n, (T*)w.W, nullptr, s)))
        return rc;
    if ((rc = ngf_terms_impl<T>(&L->img, (const T*)w.W, (const T*)L->gR, (const T*)L->nR, L->tau,
                                L->rho, (T*)w.terms, (T*)w.q, s)))
        return rc;
    if ((rc = pairwise_sum_impl<T>((const T*)w.terms, n, w.dws + 4, 1, hbar / 2, s))) return rc;
    if ((rc = gradient_t_impl<T>(&L->img, (const T*)w.q, (T*)w.s, s))) return rc;
    if ((rc = warp_jt_impl<T>(&L->img, (const T*)L->T, (const T*)w.yhat, (const T*)w.s, n,
                              (T*)w.ghat, s)))
        return rc;
    if ((rc = apply_Pt_variant_impl<T>(L->plan, L->pt_variant, (const T*)w.ghat, (T*)w.gD, s))) return rc;
    if ((rc = curvature_impl<T>(&L->def, (const T*)y, w.dws + 5, (T*)grad, (const T*)w.gD, L->alpha,
                                (T*)w.cws, w.dws, s)))
        return rc;
    NGF_LAUNCH(k_nonfinite<T>, blocks_for(3 * grid_n(L->def), 256), 256, 0, s, (const T*)y,
               3 * grid_n(L->def), L->flag);
    NGF_LAUNCH(k_finish_exact, 1, 1, 0, s, w.dws + 4, w.dws + 5, L->alpha, L->flag, scal);
    NGF_CHECK_LAUNCH();
    return 0;
}

}  // namespace ngf

using namespace ngf;

extern "C" {

static int level_create_impl(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                             const void* T, const void* R, const void* gR, const void* nR,
                             double tau, double rho, double alpha, void* stream, ngf_level_t** out,
                             int64_t zlo = 0, int64_t zhi = -1) {
    if (!out || !T || (!R && (!gR || !nR)) || (dtype != NGF_F32 && dtype != NGF_F64)) return NGF_EARG;
    if (!grid_ok(img_grid) || !grid_ok(def_grid)) return NGF_EARG;
    if (zhi < 0) zhi = img_grid->dims[2];
    if (zlo < 0 || zhi > img_grid->dims[2] || zlo >= zhi || (!R && (zlo != 0 || zhi != img_grid->dims[2])))
        return NGF_EARG;
    if (!(tau > 0) || !(rho > 0)) return NGF_EARG;
    *out = nullptr;
    ngf_level* L = (ngf_level*)std::calloc(1, sizeof(ngf_level));
    if (!L) return NGF_ENOMEM;
    if (cudaEventCreateWithFlags(&L->done, cudaEventDisableTiming) != cudaSuccess) {
        std::free(L);
        return NGF_ENOMEM;
    }
    L->dtype = dtype;
    L->img = *img_grid;
    L->def = *def_grid;
    L->T = T;
    L->tau = tau;
    L->rho = rho;
    L->alpha = alpha;
    int rc = ngf_plan_create(def_grid, img_grid, &L->plan);
    if (!rc) {
        rc = plan_upload(L->plan);
        if (rc) ngf_plan_destroy(L->plan);
    }
    if (rc) {
        std::free(L);
        return rc;
    }
    cudaStream_t s = as_stream(stream);
    const int64_t n = grid_n(L->img);
    const size_t es = dtype == NGF_F32 ? 4 : 8;
    if (dev_alloc(&L->gR, 3 * n * es) || dev_alloc(&L->nR, n * es) || dev_alloc(&L->RT, n * 4 * es) ||
        dev_alloc((void**)&L->flag, 16)) {
        ngf_level_destroy(L);
        return NGF_ENOMEM;
    }
    cudaMemsetAsync(L->flag, 0, 16, s);
    // a z-slab level (config 5) computes its reference terms on its own planes only
    L->slab_terms = zlo != 0 || zhi != L->img.dims[2];
    const int64_t plane = L->img.dims[0] * L->img.dims[1];
    if (R) {
        rc = dtype == NGF_F32
                 ? ref_terms_impl<float>(&L->img, (const float*)R, rho, (float*)L->gR, (float*)L->nR, s, zlo, zhi)
                 : ref_terms_impl<double>(&L->img, (const double*)R, rho, (double*)L->gR,
                                          (double*)L->nR, s, zlo, zhi);
    } else {
        rc = (int)cudaMemcpyAsync(L->gR, gR, 3 * n * es, cudaMemcpyDeviceToDevice, s);
        if (!rc) rc = (int)cudaMemcpyAsync(L->nR, nR, n * es, cudaMemcpyDeviceToDevice, s);
    }
    if (!rc) {
        if (dtype == NGF_F32) {
            rc = pack_rt<float>((const float*)L->gR, (const float*)L->nR, n, L->RT, s, zlo * plane, zhi * plane);
            if (!rc) rc = fused_setup<float>(L, (int)zlo, (int)zhi, s);
        } else {
            rc = pack_rt<double>((const double*)L->gR, (const double*)L->nR, n, L->RT, s, zlo * plane, zhi * plane);
            if (!rc) rc = fused_setup<double>(L, (int)zlo, (int)zhi, s);
        }
    }
    record_done(L->done, s);  // the creation kernels (reference terms, packing)
    if (rc) {
        ngf_level_destroy(L);
        return rc;
    }
    *out = L;
    return NGF_OK;
}

int ngf_level_create(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                     const void* T, const void* R, double tau, double rho, double alpha,
                     void* stream, ngf_level_t** out) {
    if (!R) return NGF_EARG;
    return level_create_impl(img_grid, def_grid, dtype, T, R, nullptr, nullptr, tau, rho, alpha,
                             stream, out);
}

int ngf_level_create_zslab(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                           const void* T, const void* R, double tau, double rho, double alpha,
                           int64_t zlo, int64_t zhi, void* stream, ngf_level_t** out) {
    if (!R) return NGF_EARG;
    return level_create_impl(img_grid, def_grid, dtype, T, R, nullptr, nullptr, tau, rho, alpha,
                             stream, out, zlo, zhi);
}

int ngf_level_create_terms(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                           const void* T, const void* gR, const void* nR, double tau, double rho,
                           double alpha, void* stream, ngf_level_t** out) {
    return level_create_impl(img_grid, def_grid, dtype, T, nullptr, gR, nR, tau, rho, alpha,
                             stream, out);
}

void ngf_level_destroy(ngf_level_t* L) {
    if (!L) return;
    // no kernel may still use the level's buffers: wait for its last launch
    if (!L->done || cudaEventSynchronize(L->done) != cudaSuccess) {
        cudaGetLastError();
        cudaDeviceSynchronize();
    }
    if (L->done) cudaEventDestroy(L->done);
    if (L->plan) {
        L->plan->idle = 1;
        ngf_plan_destroy(L->plan);
    }
    void* bufs[] = {L->flag, L->Tpad, L->gR, L->nR, L->RT, L->fp_blob, L->partial, L->dpart, L->spart,
                    L->ex.yhat, L->ex.W, L->ex.terms, L->ex.q, L->ex.s, L->ex.ghat, L->ex.gD,
                    L->ex.cws, L->ex.dws, L->hx, L->hg, L->hsc};
    for (void* b : bufs) dev_free(b);
    if (L->hsc_pin) cudaFreeHost(L->hsc_pin);
    if (L->pipe) {
        PipeState& ps = *L->pipe;
        for (int i = 0; i < kPipeMax; ++i) {
            if (ps.st[i]) cudaStreamDestroy(ps.st[i]);
            if (ps.evH[i]) cudaEventDestroy(ps.evH[i]);
            if (ps.evP[i]) cudaEventDestroy(ps.evP[i]);
            if (ps.evM[i]) cudaEventDestroy(ps.evM[i]);
        }
        if (ps.up) cudaStreamDestroy(ps.up);
        if (ps.down) cudaStreamDestroy(ps.down);
        if (ps.start) cudaEventDestroy(ps.start);
        if (ps.fin) cudaEventDestroy(ps.fin);
        delete L->pipe;
    }
    delete L->ctl;
    for (int k = 0; k < 2; ++k)
        if (L->ev[k]) cudaEventDestroy(L->ev[k]);
    std::free(L);
}

int ngf_level_eval(ngf_level_t* L, const void* y, void* grad, double* scalars_dev, int mode,
                   void* stream) {
    if (!L || !y || !grad || !scalars_dev) return NGF_EARG;
    cudaStream_t s = as_stream(stream);
    int rc;
    if (mode == 1) {
        if (L->slab_terms) return NGF_ESTATE;  // the exact path needs the full reference terms
        rc = L->dtype == NGF_F32 ? eval_exact<float>(L, y, grad, scalars_dev, s)
                                 : eval_exact<double>(L, y, grad, scalars_dev, s);
    } else if (mode == 0 || mode == 2) {
        if (L->slab_terms && mode == 0) return NGF_ESTATE;  // only the slab partial exists
        rc = fused_part(L, y, grad, scalars_dev, s, mode == 2 ? 1 : 0);
    } else {
        return NGF_EARG;
    }
    record_done(L->done, s);
    return rc;
}

}  // extern "C"

namespace ngf {

static int pipe_parts() {
    static const int n = [] {
        const char* e = std::getenv("NGF_PIPE_PARTS");
        return e ? std::max(0, std::min(kPipeMax, std::atoi(e))) : 4;
    }();
    return n;
}

static int pipe_init(ngf_level* L) {
    if (L->pipe) return 0;
    PipeState* ps = new PipeState();
    L->pipe = ps;
    int lo = 0, hi = 0;  // numerically: lo = least, hi = greatest priority
    NGF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < kPipeMax; ++i) {
        // earlier parts first: their CTAs are dispatched ahead of a later part's
        const int pr = std::min(lo, hi + i);
        NGF_CUDA(cudaStreamCreateWithPriority(&ps->st[i], cudaStreamNonBlocking, pr));
        NGF_CUDA(cudaEventCreateWithFlags(&ps->evH[i], cudaEventDisableTiming));
        NGF_CUDA(cudaEventCreateWithFlags(&ps->evP[i], cudaEventDisableTiming));
        NGF_CUDA(cudaEventCreateWithFlags(&ps->evM[i], cudaEventDisableTiming));
    }
    NGF_CUDA(cudaStreamCreateWithPriority(&ps->up, cudaStreamNonBlocking, hi));
    NGF_CUDA(cudaStreamCreateWithPriority(&ps->down, cudaStreamNonBlocking, hi));
    NGF_CUDA(cudaEventCreateWithFlags(&ps->start, cudaEventDisableTiming));
    NGF_CUDA(cudaEventCreateWithFlags(&ps->fin, cudaEventDisableTiming));
    return 0;
}

// deformation planes [a, b) of the three components between the (3, ndz, ndy, ndx) host and
// device arrays: one strided copy
static cudaError_t copy_planes(void* dst, const void* src, int64_t a, int64_t b, int64_t plane, int64_t m,
                               cudaMemcpyKind kind, cudaStream_t s) {
    if (b <= a) return cudaSuccess;
    const size_t es = sizeof(float), o = (size_t)(a * plane) * es;
    return cudaMemcpy2DAsync((char*)dst + o, (size_t)m * es, (const char*)src + o, (size_t)m * es,
                             (size_t)((b - a) * plane) * es, 3, kind, s);
}

// Returns kNotPiped when the level does not take the pipelined path (the caller runs the
// serial one); else 0 or an error.
constexpr int kNotPiped = -1000;
static int eval_host_pipelined(ngf_level* L, const void* y_host, void* grad_host, double* scalars_host,
                               cudaStream_t s) {
    if (L->dtype != NGF_F32 || L->fp.variant != kLeanVariant || !L->ctl || L->slab_terms || L->timing)
        return kNotPiped;
    const lean::Ctl& c = *L->ctl;
    const int nc = c.nchunk;
    const int P = std::min(L->pipe_req > 0 ? L->pipe_req : pipe_parts(), nc);
    if (P < 2 || !host_is_pinned(y_host) || !host_is_pinned(grad_host)) return kNotPiped;
    if (int rc = pipe_init(L)) return rc;
    PipeState& ps = *L->pipe;
    // The totals go straight into the page-locked scalars (mapped); the gradient planes of
    // the last two parts too (their post kernels' stores cross PCIe, no copy after them:
    // both finish with the march's last wave), the other parts' planes by copies as they
    // complete.  NGF_PIPE_MAPPED: 0 copies only, 1 every part mapped, 2 the last part
    // mapped, 3 (default) the last two.
    static const int map_mode = std::getenv("NGF_PIPE_MAPPED") ? std::atoi(std::getenv("NGF_PIPE_MAPPED")) : 3;
    const bool mapped_ok = map_mode != 0;
    void* g_map = nullptr;
    void* sc_map = nullptr;
    if (mapped_ok && (cudaHostGetDevicePointer(&g_map, grad_host, 0) != cudaSuccess ||
                      cudaHostGetDevicePointer(&sc_map, L->hsc_pin, 0) != cudaSuccess)) {
        cudaGetLastError();
        g_map = sc_map = nullptr;
    }
    const bool mapped = g_map && sc_map;
    const int64_t ndz = L->def.dims[2], plane = L->def.dims[0] * L->def.dims[1], m = plane * ndz;
    const int npc = (int)((ndz + kPostKZ - 1) / kPostKZ);
    const int wz = L->fp.wz;
    // parts: chunks [gb[i], gb[i+1]); deformation planes final after part i: those below the
    // next part's lowest window plane (post chunks [pc[i], pc[i+1])); y planes part i needs:
    // its chunks' windows and the post kernel's +-2 plane neighbourhood ([0, yz[i+1]))
    int gb[kPipeMax + 1], pc[kPipeMax + 1], yz[kPipeMax + 1];
    for (int i = 0; i <= P; ++i) gb[i] = (int)((int64_t)nc * i / P);
    pc[0] = 0;
    yz[0] = 0;
    for (int i = 0; i < P; ++i) {
        const bool last = i == P - 1;
        pc[i + 1] = last ? npc : std::max(pc[i], c.wzlo[gb[i + 1]] / kPostKZ);
        const int64_t need = std::max<int64_t>(c.wzlo[gb[i + 1] - 1] + wz, (int64_t)kPostKZ * pc[i + 1] + 2);
        yz[i + 1] = last ? (int)ndz : (int)std::max<int64_t>(yz[i], std::min<int64_t>(ndz, need));
    }
    static const bool trace = std::getenv("NGF_PIPE_TRACE") != nullptr;
    cudaEvent_t tev[4 * kPipeMax + 2] = {};
    int ntev = 0;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEventCreate(&tev[ntev]);
        cudaEventRecord(tev[ntev++], st);
    };
    mark(s);
    NGF_CUDA(cudaEventRecord(ps.start, s));
    NGF_CUDA(cudaStreamWaitEvent(ps.up, ps.start, 0));
    NGF_CUDA(cudaStreamWaitEvent(ps.down, ps.start, 0));
    for (int i = 0; i < P; ++i) {
        NGF_CUDA(cudaStreamWaitEvent(ps.st[i], ps.start, 0));
        NGF_CUDA(copy_planes(L->hx, y_host, yz[i], yz[i + 1], plane, m, cudaMemcpyHostToDevice, ps.up));
        NGF_CUDA(cudaEventRecord(ps.evH[i], ps.up));
        mark(ps.up);
    }
    FusedArgs<float> a = fused_args<float>(L, L->hx);
    double* sout = mapped ? (double*)sc_map : L->hsc;
    for (int i = 0; i < P; ++i) {
        cudaStream_t si = ps.st[i];
        NGF_CUDA(cudaStreamWaitEvent(si, ps.evH[i], 0));
        a.chunk0 = gb[i];
        a.nchunks = gb[i + 1] - gb[i];
        fused_march_launch(a, si);
        NGF_CHECK_LAUNCH();
        mark(si);
        NGF_CUDA(cudaEventRecord(ps.evM[i], si));
        // part i's post kernel also needs the earlier parts' marches (windows overlap across
        // a part boundary; parts may finish out of order).  The totals are formed by the
        // last post block to finish over all parts: every post block counts, and each runs
        // after the marches its part waited for, so the last one runs after all of them.
        for (int j = 0; j < i; ++j) NGF_CUDA(cudaStreamWaitEvent(si, ps.evM[j], 0));
        const bool gmap = mapped && (map_mode == 1 || i == P - 1 || (map_mode == 3 && i == P - 2));
        float* gout = gmap ? (float*)g_map : (float*)L->hg;
        if (pc[i + 1] > pc[i])
            if (int rc = fused_post_range<float>(a, L->def, L->alpha, L->spart, L->ns, L->flag, gout, sout, si, pc[i],
                                                 pc[i + 1]))
                return rc;
        NGF_CUDA(cudaEventRecord(ps.evP[i], si));
        mark(si);
        if (!gmap) {
            NGF_CUDA(cudaStreamWaitEvent(ps.down, ps.evP[i], 0));
            NGF_CUDA(copy_planes(grad_host, L->hg, (int64_t)kPostKZ * pc[i],
                                 std::min<int64_t>(ndz, (int64_t)kPostKZ * pc[i + 1]), plane, m,
                                 cudaMemcpyDeviceToHost, ps.down));
        }
    }
    if (!mapped) {
        for (int i = 0; i < P; ++i) NGF_CUDA(cudaStreamWaitEvent(ps.down, ps.evP[i], 0));
        NGF_CUDA(cudaMemcpyAsync(L->hsc_pin, L->hsc, 3 * sizeof(double), cudaMemcpyDeviceToHost, ps.down));
        NGF_CUDA(cudaEventRecord(ps.fin, ps.down));
        NGF_CUDA(cudaStreamWaitEvent(s, ps.fin, 0));
    } else {
        for (int i = 0; i < P; ++i) NGF_CUDA(cudaStreamWaitEvent(s, ps.evP[i], 0));
        NGF_CUDA(cudaEventRecord(ps.fin, ps.down));  // the copied planes
        NGF_CUDA(cudaStreamWaitEvent(s, ps.fin, 0));
    }
    mark(s);
    NGF_CUDA(cudaStreamSynchronize(s));
    std::memcpy(scalars_host, L->hsc_pin, 3 * sizeof(double));
    if (trace) {
        // per part: H2D done (all parts first), then march end, post end; then the join
        // (microseconds after start)
        std::fprintf(stderr, "pipe P=%d mapped=%d chunks", P, (int)mapped);
        for (int i = 0; i <= P; ++i) std::fprintf(stderr, " %d", gb[i]);
        std::fprintf(stderr, " | y planes");
        for (int i = 0; i <= P; ++i) std::fprintf(stderr, " %d", yz[i]);
        std::fprintf(stderr, " | post chunks");
        for (int i = 0; i <= P; ++i) std::fprintf(stderr, " %d", pc[i]);
        std::fprintf(stderr, "\n  h2d:");
        for (int k = 1; k < ntev; ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tev[0], tev[k]);
            if (k == P + 1) std::fprintf(stderr, "\n  march/post:");
            std::fprintf(stderr, " %.1f", ms * 1e3f);
        }
        std::fprintf(stderr, "\n");
        for (int k = 0; k < ntev; ++k) cudaEventDestroy(tev[k]);
    }
    return 0;
}

}  // namespace ngf

extern "C" {

int ngf_level_eval_host(ngf_level_t* L, const void* y_host, void* grad_host, double* scalars_host,
                        int mode, void* stream) {
    if (!L || !y_host || !grad_host || !scalars_host || (mode != 0 && mode != 1)) return NGF_EARG;
    cudaStream_t s = as_stream(stream);
    const size_t vb = (size_t)3 * L->def.dims[0] * L->def.dims[1] * L->def.dims[2] *
                      (L->dtype == NGF_F32 ? 4 : 8);
    if (!L->hx) {
        if (dev_alloc(&L->hx, vb) || dev_alloc(&L->hg, vb) || dev_alloc((void**)&L->hsc, 4 * sizeof(double)))
            return NGF_ENOMEM;
        NGF_CUDA(cudaHostAlloc((void**)&L->hsc_pin, 4 * sizeof(double), cudaHostAllocDefault));
        // the buffers come from the stream-ordered pool on the legacy stream: complete the
        // allocations before any other stream (the caller's, the pipeline's) touches them
        NGF_CUDA(cudaStreamSynchronize(0));
    }
    if (mode == 0) {
        const int rc = eval_host_pipelined(L, y_host, grad_host, scalars_host, s);
        if (rc != kNotPiped) {
            record_done(L->done, s);
            return rc;
        }
    }
    if (int rc = host_upload(L->hx, y_host, vb, s)) return rc;
    if (int rc = ngf_level_eval(L, L->hx, L->hg, L->hsc, mode, stream)) return rc;
    // the scalars go first: the gradient download waits for everything before it
    NGF_CUDA(cudaMemcpyAsync(L->hsc_pin, L->hsc, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (int rc = host_download(grad_host, L->hg, vb, s)) return rc;
    std::memcpy(scalars_host, L->hsc_pin, 3 * sizeof(double));
    return 0;
}

int ngf_level_add_curvature(ngf_level_t* L, const void* y, void* grad, double* scalars_dev,
                            void* stream) {
    if (!L || !y || !grad || !scalars_dev) return NGF_EARG;
    const int rc = fused_part(L, y, grad, scalars_dev, as_stream(stream), 2);
    record_done(L->done, as_stream(stream));
    return rc;
}

int ngf_level_set_host_pipeline(ngf_level_t* L, int parts) {
    if (!L || parts < 0 || parts > kPipeMax) return NGF_EARG;
    L->pipe_req = parts;
    return 0;
}

int ngf_level_set_zrange(ngf_level_t* L, int64_t zlo, int64_t zhi) {
    if (!L || zlo < 0 || zhi > L->img.dims[2] || zlo >= zhi) return NGF_EARG;
    NGF_CUDA(cudaDeviceSynchronize());
    void* bufs[] = {L->fp_blob, L->partial, L->dpart, L->spart};
    for (void* b : bufs) dev_free(b);
    L->fp_blob = L->partial = nullptr;
    L->dpart = L->spart = nullptr;
    return L->dtype == NGF_F32 ? fused_setup<float>(L, (int)zlo, (int)zhi)
                               : fused_setup<double>(L, (int)zlo, (int)zhi);
}

int ngf_level_set_pt_variant(ngf_level_t* L, int variant) {
    if (!L || variant < 0 || variant > 2) return NGF_EARG;
    L->pt_variant = variant;
    return 0;
}

int ngf_level_set_timing(ngf_level_t* L, int on) {
    if (!L) return NGF_EARG;
    if (on && !L->ev[0]) {
        NGF_CUDA(cudaEventCreate(&L->ev[0]));
        NGF_CUDA(cudaEventCreate(&L->ev[1]));
    }
    L->timing = on ? 1 : 0;
    return 0;
}

int ngf_level_kernel_ms(ngf_level_t* L, float* ms) {
    if (!L || !ms || !L->ev[0]) return NGF_ESTATE;
    NGF_CUDA(cudaEventSynchronize(L->ev[1]));
    NGF_CUDA(cudaEventElapsedTime(ms, L->ev[0], L->ev[1]));
    return 0;
}

int ngf_level_info(const ngf_level_t* L, int64_t* info) {
    // [0] CTAs of the fused kernel, [1] smem bytes, [2] z chunk, [3..5] window wx, wy, wz,
    // [6..8] tiles ntx, nty, ntz
    if (!L || !info) return NGF_EARG;
    const FusedPlan& fp = L->fp;
    int64_t v[9] = {fp.n_cta, (int64_t)fp.smem_bytes, fp.cz, fp.wx, fp.wy, fp.wz, fp.ntx, fp.nty, fp.ntz};
    for (int k = 0; k < 9; ++k) info[k] = v[k];
    return 0;
}

const void* ngf_level_ref_terms(const ngf_level_t* L) { return L ? L->RT : nullptr; }

int ngf_level_variant(const ngf_level_t* L) { return L ? L->fp.variant : NGF_EARG; }

}  // extern "C"
