// L-BFGS device vector algebra shared by the host-driven driver (solver.cu) and the
// graph-driven one (solver_graph.cu).
#pragma once

#include "common.cuh"

namespace ngf {

constexpr int kMaxMem = 32;

// Arguments of the two-loop recursion (lbfgs.py:68-91): pairs oldest first.  Passed by
// value from the host driver; the graph driver keeps one in device memory and rewrites
// S, Y, rho, gamma and m from its device-side history before every launch.
template <typename T>
struct TwoLoopArgs {
    const T* S[kMaxMem];
    const T* Y[kMaxMem];
    double rho[kMaxMem];
    double gamma;
    int m;
    const T* g;
    T* d;  // holds q during the recursion, -q at the end
    int64_t n;
    double* parts;  // [2][kRedBlocks]
    double* slope;
};

// Largest vector the register-resident cluster two-loop takes (no cooperative launch,
// so it can sit inside a conditional graph body).
constexpr int64_t kTwoLoopClusterMaxN = 16 * 512 * 16;

// Launchers with device-resident arguments (graph capture): the two-loop reads *args,
// the pair kernel writes to *s_ptr / *y_ptr, the step reads *t.
template <typename T>
int two_loop_dev_launch(const TwoLoopArgs<T>* args, int64_t n, cudaStream_t s);
// (the pair kernel's reduction scratch belongs to `owner`, the stream the graph runs on)
template <typename T>
int pair_dev_launch(const T* xn, const T* x, const T* gn, const T* g, T* const* s_ptr, T* const* y_ptr,
                    int64_t n, double* out, cudaStream_t s, cudaStream_t owner);
template <typename T>
int axpy_dev_launch(const T* x, const double* t, const T* d, T* out, int64_t n, cudaStream_t s);
// scratch partials of the reductions on `owner` (allocated on first use; call before any
// capture)
double* lbfgs_parts(cudaStream_t owner);

}  // namespace ngf
