// Device helpers of the fused evaluation kernel.
#pragma once
#include "common.cuh"
#include "eval_fused.cuh"

namespace ngf {

template <typename T>
__host__ __device__ __forceinline__ void fd_coef(int i, int n, T ih, T& cm, T& c0, T& cp) {
    // derivative at index i as cm*v[i-1] + c0*v[i] + cp*v[i+1] (warp.py:130-143)
    cm = (T)0;
    c0 = (T)0;
    cp = (T)0;
    if (n < 2 || i < 0 || i >= n) return;
    if (i == 0) {
        c0 = -ih;
        cp = ih;
    } else if (i == n - 1) {
        cm = -ih;
        c0 = ih;
    } else {
        cm = (T)-0.5 * ih;
        cp = (T)0.5 * ih;
    }
}

// transpose coefficients at index i: multiply q[i-1], q[i], q[i+1]
template <typename T>
__host__ __device__ __forceinline__ void fdt_coef(int i, int n, T ih, T& gm, T& g0, T& gp) {
    T a, b, c;
    fd_coef<T>(i - 1, n, ih, a, b, c);
    gm = c;
    fd_coef<T>(i, n, ih, a, b, c);
    g0 = b;
    fd_coef<T>(i + 1, n, ih, a, b, c);
    gp = a;
}

struct __align__(16) dbl4 {
    double x, y, z, w;
};
template <typename T> struct V4Sel;
template <> struct V4Sel<float> { using type = float4; };
template <> struct V4Sel<double> { using type = dbl4; };
template <typename T> using V4T = typename V4Sel<T>::type;

template <typename T>
struct FusedArgs {
    int nx, ny, nz, ndx, ndy, ndz;
    T ox, oy, oz;     // template (= image) grid origin, working dtype
    T hx, hy, hz;     // spacing, working dtype
    T ihx, ihy, ihz;  // 1 / spacing (derivative scale)
    int pow2x, pow2y, pow2z;  // spacing is a power of two: division == multiply by exact reciprocal
    T nm1x, nm1y, nm1z;       // n - 1: upper end of the hull test (warp.py:39)
    T hix, hiy, hiz;          // max(n - 2, 0): largest lower corner (warp.py:50)
    const int32_t *i0x, *i0y, *i0z;  // image -> def lower index (transfer.py:54-63)
    const T *w1x, *w1y, *w1z;        // dtype(w1)
    const T* Tv;                     // template values
    const V4T<T>* RT;                // packed (gR/nR, 1/nR)
    const T* y;                      // deformation (3, M)
    T* partial;                      // [n_cta][3][wz][wy][wx]
    double* dpart;                   // [n_cta]
    T tau2, taurho, neg_hbar;
    double half_hbar;
    FusedPlan fp;
    int chunk0, nchunks;  // lean march: z chunks [chunk0, chunk0 + nchunks) (nchunks 0: all)
};

__device__ __forceinline__ float lerp_exact(float a0, float a1, float w) {
    // a0 * (1 - w) + a1 * w, each op correctly rounded, no contraction (transfer.py:126)
    return __fadd_rn(__fmul_rn(a0, __fsub_rn(1.0f, w)), __fmul_rn(a1, w));
}
__device__ __forceinline__ double lerp_exact(double a0, double a1, double w) {
    return __dadd_rn(__dmul_rn(a0, __dsub_rn(1.0, w)), __dmul_rn(a1, w));
}
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float fmin_t(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double fmin_t(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float fmax_t(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double fmax_t(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float fmaf_t(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaf_t(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float rsqrt_t(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_t(double x) { return rsqrt(x); }

__device__ __forceinline__ float4 ld_rt(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ dbl4 ld_rt(const dbl4* p) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = __ldcs(q), b = __ldcs(q + 1);
    dbl4 r;
    r.x = a.x;
    r.y = a.y;
    r.z = b.x;
    r.w = b.y;
    return r;
}

// Trilinear value and derivative / h from the 8 corners c[dx + 2 dy + 4 dz] (lerp form
// of warp.py:79-85 and :111-120)
template <typename T>
__device__ __forceinline__ void trilinear(const FusedArgs<T>& a, const T (&c)[8], T fx, T fy, T fz,
                                          T& W, T& d0, T& d1, T& d2) {
    const T e00 = c[1] - c[0], e10 = c[3] - c[2], e01 = c[5] - c[4], e11 = c[7] - c[6];
    const T a00 = fmaf_t(fx, e00, c[0]), a10 = fmaf_t(fx, e10, c[2]);
    const T a01 = fmaf_t(fx, e01, c[4]), a11 = fmaf_t(fx, e11, c[6]);
    const T dy0 = a10 - a00, dy1 = a11 - a01;
    const T b0 = fmaf_t(fy, dy0, a00), b1 = fmaf_t(fy, dy1, a01);
    const T dz = b1 - b0;
    W = fmaf_t(fz, dz, b0);
    const T ex0 = fmaf_t(fy, e10 - e00, e00), ex1 = fmaf_t(fy, e11 - e01, e01);
    d0 = fmaf_t(fz, ex1 - ex0, ex0) * a.ihx;
    d1 = fmaf_t(fz, dy1 - dy0, dy0) * a.ihy;
    d2 = dz * a.ihz;
}

// NGF ratio, the distance term and q = dD/d(grad W) (ngf.py:70-112), with the
// reference terms packed as (gR/nR, 1/nR)
template <typename T>
__device__ __forceinline__ void ngf_q(const FusedArgs<T>& a, T gx, T gy, T gz, const V4T<T>& rt,
                                      T& qx, T& qy, T& qz, double& dacc) {
    const T dot = fmaf_t(gx, rt.x, fmaf_t(gy, rt.y, gz * rt.z));
    const T sq = fmaf_t(gx, gx, fmaf_t(gy, gy, fmaf_t(gz, gz, a.tau2)));
    const T inv_nt = rsqrt_t(sq);
    const T r = fmaf_t(a.taurho, rt.w, dot) * inv_nt;
    dacc += (double)fmaf_t(-r, r, (T)1);
    const T cf = a.neg_hbar * r * inv_nt;
    const T t1 = r * inv_nt;
    qx = cf * fmaf_t(-t1, gx, rt.x);
    qy = cf * fmaf_t(-t1, gy, rt.y);
    qz = cf * fmaf_t(-t1, gz, rt.z);
}

template <typename T>
int fused_eval_launch(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int ns,
                      int* flag, T* grad, double* scalars, cudaStream_t s, cudaEvent_t ev0 = nullptr,
                      cudaEvent_t ev1 = nullptr, int part = 0);
// the post-march kernel alone over post chunks [pc0, pc1) of kPostKZ deformation planes
// (the pipelined host evaluation; no programmatic dependent launch).  The block counter
// spans all post launches of the evaluation: the last block to finish forms J, D, S.
template <typename T>
int fused_post_range(const FusedArgs<T>& a, const ngf_grid_t& dg, double alpha, double* spart, int ns, int* flag,
                     T* grad, double* scalars, cudaStream_t s, int pc0, int pc1);
void fused_march_launch(const FusedArgs<float>& a, cudaStream_t s);
constexpr int kPostKZ = 4;  // deformation planes per k_post block
template <typename T> int fused_prepare(int variant, size_t smem);
template <typename T> size_t fused_smem(int variant, int wx, int wy);
void fused_variant_geom(int variant, int* ty, int* nthreads);
int fused_variant_count();
template <typename T> int pack_rt(const T* gR, const T* nR, int64_t n, void* out, cudaStream_t s,
                                  int64_t first = 0, int64_t last = -1);

}  // namespace ngf
