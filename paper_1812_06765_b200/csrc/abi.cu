// extern "C" entry points of the standalone operators (include/ngf_b200.h).

#include "common.cuh"
#include "ops_exact.cuh"

using namespace ngf;

#define NGF_DISPATCH(dtype, CALL_F32, CALL_F64)         \
    do {                                                \
        if ((dtype) == NGF_F32) return (CALL_F32);      \
        if ((dtype) == NGF_F64) return (CALL_F64);      \
        return NGF_EARG;                                \
    } while (0)

extern "C" {

int ngf_apply_P(const ngf_plan_t* p, int dtype, const void* y, void* yhat, void* stream) {
    if (!p || !y || !yhat) return NGF_EARG;
    NGF_DISPATCH(dtype, apply_P_impl<float>(p, (const float*)y, (float*)yhat, as_stream(stream)),
                 apply_P_impl<double>(p, (const double*)y, (double*)yhat, as_stream(stream)));
}

int ngf_apply_Pt(const ngf_plan_t* p, int dtype, const void* r, void* out, void* stream) {
    if (!p || !r || !out) return NGF_EARG;
    NGF_DISPATCH(dtype, apply_Pt_impl<float>(p, (const float*)r, (float*)out, as_stream(stream)),
                 apply_Pt_impl<double>(p, (const double*)r, (double*)out, as_stream(stream)));
}

int ngf_apply_Pt_variant(const ngf_plan_t* p, int dtype, int variant, const void* r, void* out,
                         void* stream) {
    if (!p || !r || !out) return NGF_EARG;
    NGF_DISPATCH(dtype,
                 apply_Pt_variant_impl<float>(p, variant, (const float*)r, (float*)out, as_stream(stream)),
                 apply_Pt_variant_impl<double>(p, variant, (const double*)r, (double*)out, as_stream(stream)));
}

int ngf_sample_field(const ngf_grid_t* g, int dtype, const void* y, const double* pts, int64_t n, double* out,
                     void* stream) {
    if (!grid_ok(g) || !y || (n > 0 && (!pts || !out)) || n < 0) return NGF_EARG;
    NGF_DISPATCH(dtype, sample_field_impl<float>(g, (const float*)y, pts, n, out, as_stream(stream)),
                 sample_field_impl<double>(g, (const double*)y, pts, n, out, as_stream(stream)));
}

int ngf_warp(const ngf_grid_t* tg, int dtype, const void* T, const void* yhat, int64_t n, void* W,
             uint8_t* mask, void* stream) {
    if (!grid_ok(tg) || !T || !yhat || !W || n < 0) return NGF_EARG;
    if (n == 0) return 0;
    NGF_DISPATCH(dtype,
                 warp_impl<float>(tg, (const float*)T, (const float*)yhat, n, (float*)W, mask,
                                  as_stream(stream)),
                 warp_impl<double>(tg, (const double*)T, (const double*)yhat, n, (double*)W, mask,
                                   as_stream(stream)));
}

int ngf_warp_jt(const ngf_grid_t* tg, int dtype, const void* T, const void* yhat, const void* s,
                int64_t n, void* out, void* stream) {
    if (!grid_ok(tg) || !T || !yhat || !s || !out || n < 0) return NGF_EARG;
    if (n == 0) return 0;
    NGF_DISPATCH(dtype,
                 warp_jt_impl<float>(tg, (const float*)T, (const float*)yhat, (const float*)s, n,
                                     (float*)out, as_stream(stream)),
                 warp_jt_impl<double>(tg, (const double*)T, (const double*)yhat, (const double*)s, n,
                                      (double*)out, as_stream(stream)));
}

int ngf_gradient(const ngf_grid_t* g, int dtype, const void* v, void* out3, void* stream) {
    if (!grid_ok(g) || !v || !out3) return NGF_EARG;
    NGF_DISPATCH(dtype, gradient_impl<float>(g, (const float*)v, (float*)out3, as_stream(stream)),
                 gradient_impl<double>(g, (const double*)v, (double*)out3, as_stream(stream)));
}

int ngf_gradient_t(const ngf_grid_t* g, int dtype, const void* w3, void* out, void* stream) {
    if (!grid_ok(g) || !w3 || !out) return NGF_EARG;
    NGF_DISPATCH(dtype, gradient_t_impl<float>(g, (const float*)w3, (float*)out, as_stream(stream)),
                 gradient_t_impl<double>(g, (const double*)w3, (double*)out, as_stream(stream)));
}

int ngf_ref_terms(const ngf_grid_t* g, int dtype, const void* R, double rho, void* gR3, void* nR,
                  void* stream) {
    if (!grid_ok(g) || !R || !gR3 || !nR || !(rho > 0)) return NGF_EARG;
    NGF_DISPATCH(dtype,
                 ref_terms_impl<float>(g, (const float*)R, rho, (float*)gR3, (float*)nR,
                                       as_stream(stream)),
                 ref_terms_impl<double>(g, (const double*)R, rho, (double*)gR3, (double*)nR,
                                        as_stream(stream)));
}

int ngf_ngf_terms(const ngf_grid_t* g, int dtype, const void* W, const void* gR3, const void* nR,
                  double tau, double rho, void* terms, void* q3, void* stream) {
    if (!grid_ok(g) || !W || !gR3 || !nR || !(tau > 0) || !(rho > 0)) return NGF_EARG;
    NGF_DISPATCH(dtype,
                 ngf_terms_impl<float>(g, (const float*)W, (const float*)gR3, (const float*)nR, tau,
                                       rho, (float*)terms, (float*)q3, as_stream(stream)),
                 ngf_terms_impl<double>(g, (const double*)W, (const double*)gR3, (const double*)nR,
                                        tau, rho, (double*)terms, (double*)q3, as_stream(stream)));
}

int ngf_pairwise_sum(int dtype, const void* x, int64_t n, double* out_dev, void* stream) {
    if (!out_dev || n < 0 || (n > 0 && !x)) return NGF_EARG;
    NGF_DISPATCH(dtype,
                 pairwise_sum_impl<float>((const float*)x, n, out_dev, 0, 0.0, as_stream(stream)),
                 pairwise_sum_impl<double>((const double*)x, n, out_dev, 0, 0.0, as_stream(stream)));
}

int ngf_laplacian(const ngf_grid_t* g, int dtype, const void* u, void* out, void* stream) {
    if (!grid_ok(g) || !u || !out) return NGF_EARG;
    NGF_DISPATCH(dtype, laplacian_impl<float>(g, (const float*)u, (float*)out, 1, as_stream(stream)),
                 laplacian_impl<double>(g, (const double*)u, (double*)out, 1, as_stream(stream)));
}

int ngf_laplacian_t(const ngf_grid_t* g, int dtype, const void* w, void* out, void* stream) {
    if (!grid_ok(g) || !w || !out) return NGF_EARG;
    NGF_DISPATCH(dtype,
                 laplacian_t_impl<float>(g, (const float*)w, (float*)out, 1, 1.0f, 0, nullptr, 0.0f,
                                         as_stream(stream)),
                 laplacian_t_impl<double>(g, (const double*)w, (double*)out, 1, 1.0, 0, nullptr, 0.0,
                                          as_stream(stream)));
}

int ngf_curvature(const ngf_grid_t* g, int dtype, const void* y, double* S_dev, void* grad,
                  void* stream) {
    if (!grid_ok(g) || !y) return NGF_EARG;
    const int64_t m = grid_n(*g);
    const size_t es = dtype == NGF_F64 ? 8 : 4;
    void* ws = nullptr;
    double* wd = nullptr;
    cudaStream_t s = as_stream(stream);
    NGF_CUDA(cudaMallocAsync(&ws, 6 * m * es, s));
    NGF_CUDA(cudaMallocAsync((void**)&wd, 8 * sizeof(double), s));
    int rc;
    if (dtype == NGF_F32)
        rc = curvature_impl<float>(g, (const float*)y, S_dev, (float*)grad, nullptr, 1.0,
                                   (float*)ws, wd, s);
    else if (dtype == NGF_F64)
        rc = curvature_impl<double>(g, (const double*)y, S_dev, (double*)grad, nullptr, 1.0,
                                    (double*)ws, wd, s);
    else
        rc = NGF_EARG;
    cudaFreeAsync(ws, s);
    cudaFreeAsync(wd, s);
    return rc;
}

int ngf_downsample(const ngf_grid_t* g, int dtype, const void* in, void* out, void* stream) {
    if (!grid_ok(g) || !in || !out) return NGF_EARG;
    NGF_DISPATCH(dtype, downsample_impl<float>(g, (const float*)in, (float*)out, as_stream(stream)),
                 downsample_impl<double>(g, (const double*)in, (double*)out, as_stream(stream)));
}

int ngf_prolong(const ngf_plan_t* p, int dtype, const void* yc, void* yf, void* stream) {
    if (!p || !yc || !yf) return NGF_EARG;
    ngf_plan_t* mp = const_cast<ngf_plan_t*>(p);
    if (!mp->done) NGF_CUDA(cudaEventCreateWithFlags(&mp->done, cudaEventDisableTiming));
    int rc;
    if (dtype == NGF_F32)
        rc = prolong_impl<float>(p, (const float*)yc, (float*)yf, as_stream(stream));
    else if (dtype == NGF_F64)
        rc = prolong_impl<double>(p, (const double*)yc, (double*)yf, as_stream(stream));
    else
        return NGF_EARG;
    record_done(mp->done, as_stream(stream));
    return rc;
}

}  // extern "C"
