// Declarations of the bit-exact operator implementations (ops_exact.cu).
#pragma once
#include "common.cuh"

namespace ngf {

template <typename T> int apply_P_impl(const ngf_plan_t*, const T*, T*, cudaStream_t);
template <typename T> int apply_Pt_impl(const ngf_plan_t*, const T*, T*, cudaStream_t);
// variant 0 gather, 1 scatter (atomics), 2 red-black (transfer.py:199-256)
template <typename T> int apply_Pt_variant_impl(const ngf_plan_t*, int, const T*, T*, cudaStream_t);
template <typename T>
int warp_impl(const ngf_grid_t*, const T*, const T*, int64_t, T*, uint8_t*, cudaStream_t);
template <typename T>
int warp_jt_impl(const ngf_grid_t*, const T*, const T*, const T*, int64_t, T*, cudaStream_t);
template <typename T> int gradient_impl(const ngf_grid_t*, const T*, T*, cudaStream_t);
template <typename T> int gradient_t_impl(const ngf_grid_t*, const T*, T*, cudaStream_t);
template <typename T>
int ref_terms_impl(const ngf_grid_t*, const T*, double, T*, T*, cudaStream_t, int64_t zlo = 0,
                   int64_t zhi = -1);
template <typename T>
int ngf_terms_impl(const ngf_grid_t*, const T*, const T*, const T*, double, double, T*, T*,
                   cudaStream_t);
// mode 0: *out = sum; mode 1: *out = T(scale) * sum (NEP-50 python-float times numpy scalar)
template <typename T>
int pairwise_sum_impl(const T*, int64_t, double*, int mode, double scale, cudaStream_t);
template <typename T> int laplacian_impl(const ngf_grid_t*, const T*, T*, int, cudaStream_t);
template <typename T>
int laplacian_t_impl(const ngf_grid_t*, const T*, T*, int, T, int, const T*, T, cudaStream_t);
// workspace ws: 6*M values of T; ws_d: 3 doubles
template <typename T>
int curvature_impl(const ngf_grid_t*, const T*, double*, T*, const T*, double, T*, double*,
                   cudaStream_t);
template <typename T> int downsample_impl(const ngf_grid_t*, const T*, T*, cudaStream_t);
template <typename T> int prolong_impl(const ngf_plan_t*, const T*, T*, cudaStream_t);
template <typename T>
int sample_field_impl(const ngf_grid_t*, const T*, const double*, int64_t, double*, cudaStream_t);

}  // namespace ngf
