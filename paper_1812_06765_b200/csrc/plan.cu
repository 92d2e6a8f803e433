// Grid-transfer plans: host f64 computation (bit-exact with the reference) + device upload.
//
// Reference: transfer.py:42-51 (check_compatible), :54-63 (_axis_transfer),
// :82-110 (_build_axis_plan / build_gather_plan), geometry.py:68-70 (axis_centers),
// geometry.py:92-101 (same_extent).  This translation unit is compiled with
// -Xcompiler -ffp-contract=off so the IEEE double expressions are evaluated exactly
// as numpy evaluates them (one rounding per operation, no FMA).

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace ngf {

std::atomic<int64_t> g_launches{0};

// Device memory of plans and levels comes from the device's stream-ordered pool
// (cudaMallocAsync on the legacy default stream), configured once per device to keep
// freed blocks: the levels of the next registration reuse them without driver calls
// (a 256^3 level needs ~0.6 GB).
int dev_alloc(void** ptr, size_t bytes) {
    static std::atomic<uint64_t> ready{0};
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return NGF_ENOMEM;
    if (d < 64 && !(ready.load() & (1ull << d))) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        ready.fetch_or(1ull << d);
    }
    *ptr = nullptr;
    if (bytes == 0) bytes = 1;
    return cudaMallocAsync(ptr, bytes, 0) == cudaSuccess ? NGF_OK : NGF_ENOMEM;
}

void dev_free(void* ptr) {
    if (ptr) cudaFreeAsync(ptr, 0);
}

int upload_blocking(void* dst, const void* src, size_t bytes) {
    NGF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, 0));
    NGF_CUDA(cudaStreamSynchronize(0));
    return 0;
}

static bool same_extent(const ngf_grid_t& a, const ngf_grid_t& b, double tol = 1e-9) {
    for (int k = 0; k < 3; ++k) {
        double lo_a = a.origin[k] - a.spacing[k] / 2;
        double lo_b = b.origin[k] - b.spacing[k] / 2;
        if (std::fabs(lo_a - lo_b) > tol) return false;
        double ext_a = (double)a.dims[k] * a.spacing[k];
        double ext_b = (double)b.dims[k] * b.spacing[k];
        if (std::fabs(lo_a + ext_a - (lo_b + ext_b)) > tol) return false;
    }
    return true;
}

// (i0, w1) per image index along axis k (transfer.py:54-63).
static void axis_transfer(const ngf_grid_t& img, const ngf_grid_t& def, int k,
                          std::vector<int32_t>& i0, std::vector<double>& w1) {
    const int64_t ni = img.dims[k];
    const int64_t nd = def.dims[k];
    i0.assign(ni, 0);
    w1.assign(ni, 0.0);
    if (nd == 1) return;
    for (int64_t i = 0; i < ni; ++i) {
        volatile double x = img.origin[k] + img.spacing[k] * (double)i;  // axis_centers
        volatile double t = (x - def.origin[k]) / def.spacing[k];
        double f = std::floor(t);
        int64_t lo = (int64_t)f;
        if (f < -1e18) lo = INT64_MIN / 2;
        if (lo < 0) lo = 0;
        if (lo > nd - 2) lo = nd - 2;
        double w = t - (double)lo;
        if (w < 0.0) w = 0.0;
        if (w > 1.0) w = 1.0;
        i0[i] = (int32_t)lo;
        w1[i] = w;
    }
}

// Transposed 1-D interpolation rows per def index (transfer.py:82-101).
static void axis_plan(const std::vector<int32_t>& i0, const std::vector<double>& w1, int nd,
                      std::vector<int32_t>& start, std::vector<int32_t>& counts,
                      std::vector<double>& weights, int& width) {
    const int ni = (int)i0.size();
    start.assign(nd, 0);
    counts.assign(nd, 0);
    for (int d = 0; d < nd; ++d) {
        int lo = 0, hi = ni;
        if (d != 0) {  // searchsorted(i0, d-1, side="left")
            lo = 0;
            while (lo < ni && i0[lo] < d - 1) ++lo;
        }
        if (d != nd - 1) {  // searchsorted(i0, d, side="right")
            hi = 0;
            while (hi < ni && i0[hi] <= d) ++hi;
        }
        start[d] = lo;
        counts[d] = hi - lo;
    }
    width = 1;
    for (int d = 0; d < nd; ++d) width = counts[d] > width ? counts[d] : width;
    weights.assign((size_t)nd * width, 0.0);
    for (int d = 0; d < nd; ++d) {
        for (int j = 0; j < counts[d]; ++j) {
            int idx = start[d] + j;
            double w = 0.0;
            if (i0[idx] == d)
                w = 1.0 - w1[idx];
            else if (i0[idx] == d - 1)
                w = w1[idx];
            weights[(size_t)d * width + j] = w;
        }
    }
}

static int build_plan(const ngf_grid_t* def_grid, const ngf_grid_t* img_grid, bool check_dims,
                      ngf_plan_t** out) {
    if (!out || !grid_ok(def_grid) || !grid_ok(img_grid)) return NGF_EARG;
    *out = nullptr;
    if (!same_extent(*def_grid, *img_grid)) return NGF_EGRID;
    if (check_dims)
        for (int k = 0; k < 3; ++k)
            if (img_grid->dims[k] < def_grid->dims[k]) return NGF_EGRID;

    ngf_plan_t* p = (ngf_plan_t*)std::calloc(1, sizeof(ngf_plan_t));
    if (!p) return NGF_ENOMEM;
    p->def_grid = *def_grid;
    p->img_grid = *img_grid;

    std::vector<int32_t> i0[3], st[3], cnt[3];
    std::vector<double> w1[3], wt[3];
    for (int k = 0; k < 3; ++k) {
        axis_transfer(*img_grid, *def_grid, k, i0[k], w1[k]);
        axis_plan(i0[k], w1[k], (int)def_grid->dims[k], st[k], cnt[k], wt[k], p->width[k]);
        p->n_img[k] = (int)img_grid->dims[k];
        p->n_def[k] = (int)def_grid->dims[k];
        int ni = p->n_img[k], nd = p->n_def[k], w = p->width[k];
        p->h_i0[k] = (int32_t*)std::malloc(ni * 4);
        p->h_w1[k] = (double*)std::malloc(ni * 8);
        p->h_start[k] = (int32_t*)std::malloc(nd * 4);
        p->h_counts[k] = (int32_t*)std::malloc(nd * 4);
        p->h_w[k] = (double*)std::malloc((size_t)nd * w * 8);
        std::memcpy(p->h_i0[k], i0[k].data(), ni * 4);
        std::memcpy(p->h_w1[k], w1[k].data(), ni * 8);
        std::memcpy(p->h_start[k], st[k].data(), nd * 4);
        std::memcpy(p->h_counts[k], cnt[k].data(), nd * 4);
        std::memcpy(p->h_w[k], wt[k].data(), (size_t)nd * w * 8);
    }
    *out = p;  // device copies are uploaded on first device use (plan_upload)
    return NGF_OK;
}

// Upload the plan's device arrays and P^T workspace (once; host-only users never pay it).
int plan_upload(ngf_plan_t* p) {
    if (p->d_blob) return NGF_OK;
    auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
    size_t blob = 0;
    for (int k = 0; k < 3; ++k) {
        size_t ni = p->n_img[k], nd = p->n_def[k], w = p->width[k];
        blob += align(ni * 4) + align(ni * 4) + align(ni * 8) + align(nd * 4) + align(nd * w * 4) +
                align(nd * w * 8);
    }
    std::vector<char> host(blob);
    void* d_blob = nullptr;
    if (dev_alloc(&d_blob, blob)) return NGF_ENOMEM;
    size_t off = 0;
    char* dbase = (char*)d_blob;
    for (int k = 0; k < 3; ++k) {
        int ni = p->n_img[k], nd = p->n_def[k], w = p->width[k];
        AxisDev& a = p->axes[k];
        a.ni = ni;
        a.nd = nd;
        a.width = w;
        auto put = [&](const void* src, size_t bytes) {
            std::memcpy(host.data() + off, src, bytes);
            void* d = dbase + off;
            off += align(bytes);
            return d;
        };
        std::vector<float> w1f(ni), wf((size_t)nd * w);
        for (int i = 0; i < ni; ++i) w1f[i] = (float)p->h_w1[k][i];
        for (size_t i = 0; i < wf.size(); ++i) wf[i] = (float)p->h_w[k][i];
        a.i0 = (const int32_t*)put(p->h_i0[k], (size_t)ni * 4);
        a.w1f = (const float*)put(w1f.data(), (size_t)ni * 4);
        a.w1d = (const double*)put(p->h_w1[k], (size_t)ni * 8);
        a.start = (const int32_t*)put(p->h_start[k], (size_t)nd * 4);
        a.wf = (const float*)put(wf.data(), wf.size() * 4);
        a.wd = (const double*)put(p->h_w[k], (size_t)nd * w * 8);
    }
    if (upload_blocking(d_blob, host.data(), blob) != 0) {
        dev_free(d_blob);
        return NGF_ENOMEM;
    }
    p->tmp_bytes = (size_t)3 * p->img_grid.dims[2] * p->def_grid.dims[1] * p->def_grid.dims[0] * 8;
    if (dev_alloc(&p->d_tmp, p->tmp_bytes)) {
        dev_free(d_blob);
        return NGF_ENOMEM;
    }
    p->d_blob = d_blob;
    return NGF_OK;
}

}  // namespace ngf

extern "C" {

int ngf_plan_create(const ngf_grid_t* def_grid, const ngf_grid_t* img_grid, ngf_plan_t** out) {
    return ngf::build_plan(def_grid, img_grid, true, out);
}

int ngf_plan_create_prolong(const ngf_grid_t* coarse, const ngf_grid_t* fine, ngf_plan_t** out) {
    return ngf::build_plan(coarse, fine, false, out);
}

void ngf_plan_destroy(ngf_plan_t* p) {
    if (!p) return;
    for (int k = 0; k < 3; ++k) {
        std::free(p->h_i0[k]);
        std::free(p->h_w1[k]);
        std::free(p->h_start[k]);
        std::free(p->h_counts[k]);
        std::free(p->h_w[k]);
    }
    if ((p->d_blob || p->d_tmp) && !p->idle) {  // no kernel may still use them
        if (!p->done || cudaEventSynchronize(p->done) != cudaSuccess) {
            cudaGetLastError();
            cudaDeviceSynchronize();
        }
    }
    if (p->done) cudaEventDestroy(p->done);
    ngf::dev_free(p->d_blob);
    ngf::dev_free(p->d_tmp);
    std::free(p);
}

int ngf_plan_axis(const ngf_plan_t* p, int axis, int32_t* host_i0, double* host_w1,
                  int32_t* host_start, int32_t* host_counts, double* host_weights,
                  int32_t* width) {
    if (!p || axis < 0 || axis > 2) return NGF_EARG;
    int ni = p->n_img[axis], nd = p->n_def[axis], w = p->width[axis];
    if (width) *width = w;
    if (host_i0) std::memcpy(host_i0, p->h_i0[axis], ni * 4);
    if (host_w1) std::memcpy(host_w1, p->h_w1[axis], ni * 8);
    if (host_start) std::memcpy(host_start, p->h_start[axis], nd * 4);
    if (host_counts) std::memcpy(host_counts, p->h_counts[axis], nd * 4);
    if (host_weights) std::memcpy(host_weights, p->h_w[axis], (size_t)nd * w * 8);
    return NGF_OK;
}

int ngf_version(void) { return 100; }

int64_t ngf_launch_count(void) { return ngf::g_launches.load(); }

const char* ngf_error_string(int code) {
    switch (code) {
        case NGF_OK: return "ok";
        case NGF_EARG: return "invalid argument";
        case NGF_EGRID: return "grid mismatch";
        case NGF_ENOMEM: return "out of memory";
        case NGF_ESTATE: return "invalid state";
        default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "unknown error";
    }
}

}  // extern "C"
