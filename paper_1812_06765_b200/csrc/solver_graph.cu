// The L-BFGS iteration loop of one level as ONE CUDA graph with device-side control
// (conditional WHILE / IF nodes, CUDA 12.4+): the decisions of ngf_lbfgs_run_level
// (solver.cu, mirroring lbfgs.py:94-181) run in single-thread control kernels between the
// evaluation, two-loop, step and pair kernels, and set the graph's condition handles, so a
// whole level runs without a host round trip.  Opt-in (ngf_lbfgs_set_graph(1)): measured
// on the 4-level 256^3 registration, the graph run of the 64^3 level takes 7.6 ms against
// ~8.6 ms for the host-driven loop, but capture + instantiation cost ~0.5 ms per level and
// the device work per iteration (evaluation, two-loop, pair, ~1.5 us per graph node) stays,
// so a registration is not faster; it becomes the better loop once a level's graph is
// reused (same level, several solves).
//
// The control kernels compute every double expression of the host driver with explicit
// round-to-nearest intrinsics (no FMA contraction), so the device decisions equal the host
// ones: the trace equals the host-driven and Python drivers' (tests/test_gpu_register.py).
// Accepted iterates and gradients move by device copies (graph node arguments are fixed).
//
// Graph (one launch per level):
//   WHILE h_iter {
//     two_loop(d) ; t = t0 ; xn = x + t d ; eval(xn) ; ctl_first        -- slope >= 0 ?
//     IF h_sd { two_loop(m = 0) ; xn = x + t d ; eval(xn) ; ctl_sd }     -- safeguard
//     ctl_ls_cond
//     WHILE h_ls { t *= shrink ; xn = x + t d ; eval(xn) ; ctl_ls }      -- Armijo backtracking
//     ctl_post_ls                                                         -- accepted ?
//     IF h_ok {
//       WHILE h_exp { xt = x + (t / shrink) d ; eval(xt) ; ctl_exp ; copy_if(xt -> xn) }
//       pair(xn - x, gn - g) ; ctl_end (history, record, stopping tests) ; x <- xn ; g <- gn
//     }
//   }

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lbfgs.cuh"

namespace ngf {

namespace {

constexpr int kSlots = kMaxMem + 2;

struct GCfg {
    double c1, shrink, t0, tol_J, tol_grad, tol_step;
    int max_ls, memory, max_iter, min_iter, max_rows;
};

template <typename T>
struct GState {
    GCfg cfg;
    double J, Jn, t, t_try, slope, g0_inf, x_scale;
    int evals, ls_evals, iter, rejected, stop, ls_failed, nrows, exp_acc, trips;
    // history: hist[0 .. hcnt) slot ids, oldest first; free slot ids in freel[0 .. nfree)
    int hcnt, nfree, cur_slot;
    int hist[kSlots], freel[kSlots];
    double sy[kSlots], yy[kSlots];
    T* slot_s[kSlots];
    T* slot_y[kSlots];
    T* cur_s;
    T* cur_y;
    double* rows;         // [max_rows][3]
    double* rec;          // [max_iter][4]
    const double* scal;   // (J, D, S, slope)
    const double* stats;  // (s.y, s.s, y.y, max|g_new|)
    TwoLoopArgs<T>* tl;
    cudaGraphConditionalHandle h_iter, h_sd, h_ls, h_ok, h_exp;
};

template <typename T>
__device__ void build_tl(GState<T>* st) {
    TwoLoopArgs<T>* tl = st->tl;
    const int m = st->hcnt;
    for (int k = 0; k < m; ++k) {
        const int j = st->hist[k];
        tl->S[k] = st->slot_s[j];
        tl->Y[k] = st->slot_y[j];
        tl->rho[k] = __ddiv_rn(1.0, st->sy[j]);
    }
    tl->gamma = m ? __ddiv_rn(st->sy[st->hist[m - 1]], st->yy[st->hist[m - 1]]) : 1.0;
    tl->m = m;
}

template <typename T>
__device__ void clear_history(GState<T>* st) {
    for (int k = 0; k < st->hcnt; ++k) st->freel[st->nfree++] = st->hist[k];
    st->hcnt = 0;
}

template <typename T>
__device__ void drop_oldest(GState<T>* st) {
    st->freel[st->nfree++] = st->hist[0];
    for (int k = 1; k < st->hcnt; ++k) st->hist[k - 1] = st->hist[k];
    --st->hcnt;
}

template <typename T>
__device__ void row(GState<T>* st) {
    if (st->nrows < st->cfg.max_rows) {
        st->rows[3 * st->nrows] = st->scal[0];
        st->rows[3 * st->nrows + 1] = st->scal[1];
        st->rows[3 * st->nrows + 2] = st->scal[2];
    }
    ++st->nrows;
}

// Jv <= J + c1 * t * slope, evaluated like the host: ((c1 * t) * slope) + J
template <typename T>
__device__ bool armijo(const GState<T>* st, double Jv, double t) {
    return isfinite(Jv) && Jv <= __dadd_rn(st->J, __dmul_rn(__dmul_rn(st->cfg.c1, t), st->slope));
}

template <typename T>
__global__ void k_ctl_begin(GState<T>* st) {
    // defensive trip count: the loop cannot outlive max_iterations even if a control
    // kernel were skipped
    if (++st->trips > st->cfg.max_iter + 1) {
        st->stop = NGF_STOP_MAX_ITER;
        cudaGraphSetConditional(st->h_iter, 0);
    }
    st->t = st->cfg.t0;
}

template <typename T>
__global__ void k_ctl_first(GState<T>* st) {
    ++st->evals;
    st->Jn = st->scal[0];
    st->slope = st->scal[3];
    st->ls_evals = 1;
    if (st->slope >= 0) {  // steepest-descent safeguard (lbfgs.py:113-116)
        --st->evals;       // the optimistic trial is discarded
        clear_history(st);
        build_tl(st);
        cudaGraphSetConditional(st->h_sd, 1);
    } else {
        cudaGraphSetConditional(st->h_sd, 0);
    }
}

template <typename T>
__global__ void k_ctl_sd(GState<T>* st) {
    ++st->evals;
    st->Jn = st->scal[0];
    st->slope = st->scal[3];
}

template <typename T>
__global__ void k_ctl_ls_cond(GState<T>* st) {
    row(st);
    cudaGraphSetConditional(st->h_ls, !armijo(st, st->Jn, st->t) && st->ls_evals < st->cfg.max_ls);
}

template <typename T>
__global__ void k_ctl_shrink(GState<T>* st) {
    st->t = __dmul_rn(st->t, st->cfg.shrink);
}

template <typename T>
__global__ void k_ctl_ls(GState<T>* st) {
    ++st->evals;
    st->Jn = st->scal[0];
    row(st);
    ++st->ls_evals;
    cudaGraphSetConditional(st->h_ls, !armijo(st, st->Jn, st->t) && st->ls_evals < st->cfg.max_ls);
}

template <typename T>
__global__ void k_ctl_post_ls(GState<T>* st) {
    if (!armijo(st, st->Jn, st->t)) {
        st->stop = NGF_STOP_LINE_SEARCH;
        st->ls_failed = 1;
        cudaGraphSetConditional(st->h_ok, 0);
        cudaGraphSetConditional(st->h_iter, 0);
        return;
    }
    cudaGraphSetConditional(st->h_ok, 1);
    const bool exp = (st->t == st->cfg.t0) && st->ls_evals < st->cfg.max_ls;
    if (exp) st->t_try = __ddiv_rn(st->t, st->cfg.shrink);
    cudaGraphSetConditional(st->h_exp, exp);
}

template <typename T>
__global__ void k_ctl_exp(GState<T>* st) {
    ++st->evals;
    const double Jt = st->scal[0];
    row(st);
    ++st->ls_evals;
    int cont = 0;
    if (armijo(st, Jt, st->t_try) && Jt < st->Jn) {
        st->t = st->t_try;
        st->Jn = Jt;
        st->exp_acc = 1;
        cont = st->ls_evals < st->cfg.max_ls;
        if (cont) st->t_try = __ddiv_rn(st->t, st->cfg.shrink);
    } else {
        st->exp_acc = 0;
    }
    cudaGraphSetConditional(st->h_exp, cont);
}

// accepted expansion trial: (xt, gt) -> (xn, gn)
template <typename T>
__global__ void k_copy_if(const GState<T>* st, const T* __restrict__ xt, const T* __restrict__ gt,
                          T* __restrict__ xn, T* __restrict__ gn, int64_t n) {
    if (!st->exp_acc) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        xn[i] = xt[i];
        gn[i] = gt[i];
    }
}

template <typename T>
__global__ void k_ctl_pair_pre(GState<T>* st) {
    const int j = st->freel[--st->nfree];
    st->cur_slot = j;
    st->cur_s = st->slot_s[j];
    st->cur_y = st->slot_y[j];
}

template <typename T>
__global__ void k_ctl_end(GState<T>* st) {
    const double sy = st->stats[0], ss = st->stats[1], yy = st->stats[2], g_inf = st->stats[3];
    const int j = st->cur_slot;
    st->sy[j] = sy;
    st->yy[j] = yy;
    const GCfg& c = st->cfg;
    if (sy > __dmul_rn(__dmul_rn(1e-10, __dsqrt_rn(ss)), __dsqrt_rn(yy))) {
        st->hist[st->hcnt++] = j;
        if (st->hcnt > c.memory) drop_oldest(st);
        st->rejected = 0;
    } else {
        st->freel[st->nfree++] = j;
        ++st->rejected;
        if (st->hcnt) drop_oldest(st);
        if (st->rejected >= c.memory) clear_history(st);
    }
    const double step_norm = __dsqrt_rn(ss);
    const double J_prev = st->J;
    st->J = st->Jn;
    const int it = st->iter;
    st->rec[4 * it] = st->J;
    st->rec[4 * it + 1] = g_inf;
    st->rec[4 * it + 2] = st->t;
    st->rec[4 * it + 3] = st->ls_evals;
    st->iter = it + 1;
    int cont = 1;
    if (it + 1 >= c.min_iter) {
        if (fabs(__dsub_rn(J_prev, st->J)) <= __dmul_rn(c.tol_J, fmax(fabs(J_prev), 1e-30))) {
            st->stop = NGF_STOP_OBJECTIVE;
            cont = 0;
        } else if (g_inf <= __dmul_rn(c.tol_grad, st->g0_inf)) {
            st->stop = NGF_STOP_GRADIENT;
            cont = 0;
        } else if (step_norm <= __dmul_rn(c.tol_step, st->x_scale)) {
            st->stop = NGF_STOP_STEP;
            cont = 0;
        }
    }
    if (cont && it + 1 == c.max_iter) {
        st->stop = NGF_STOP_MAX_ITER;
        cont = 0;
    }
    if (st->trips > c.max_iter) cont = 0;  // defensive bound (see k_ctl_begin)
    build_tl(st);
    cudaGraphSetConditional(st->h_iter, cont);
}

// ---- graph construction helpers

struct Streams {
    cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
    ~Streams() {
        for (auto x : s)
            if (x) cudaStreamDestroy(x);
    }
};

// While capturing on cs, append a conditional node and return its body graph.
int add_cond(cudaStream_t cs, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
             cudaGraph_t* body) {
    cudaStreamCaptureStatus status;
    unsigned long long id;
    cudaGraph_t g;
    const cudaGraphNode_t* deps;
    size_t nd;
    NGF_CUDA(cudaStreamGetCaptureInfo(cs, &status, &id, &g, &deps, &nd));
    if (status != cudaStreamCaptureStatusActive) return NGF_ESTATE;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    NGF_CUDA(cudaGraphAddNode(&node, g, deps, nd, &p));
    *body = p.conditional.phGraph_out[0];
    NGF_CUDA(cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies));
    return 0;
}

#define GRUN(call)              \
    do {                        \
        rc = (call);            \
        if (rc) return rc;      \
    } while (0)

}  // namespace

template <typename T>
int run_level_graph(ngf_level_t* level, int exact, T* x, T* g, T* d, T* xn, T* gn, T* xt, T* gt,
                    double* scal, double* stats, int64_t n, const ngf_lbfgs_cfg_t* cfg, double J,
                    double g0_inf, double x_scale, int evals0, int nrows0, const double* row0,
                    ngf_lbfgs_result_t* res, double* rec, double* rows, int max_rows, cudaStream_t s,
                    std::vector<void*>& owned, bool& launched) {
    int rc = 0;
    launched = false;
    if (n > kTwoLoopClusterMaxN || cfg->memory + 1 > kSlots) return NGF_EARG;
    double* parts = lbfgs_parts(s);
    if (!parts) return NGF_ENOMEM;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (dev_alloc(&p, bytes)) return nullptr;
        owned.push_back(p);
        return p;
    };
    GState<T>* dst = (GState<T>*)alloc(sizeof(GState<T>));
    TwoLoopArgs<T>* dtl = (TwoLoopArgs<T>*)alloc(sizeof(TwoLoopArgs<T>));
    double* drows = (double*)alloc((size_t)max_rows * 3 * sizeof(double));
    double* drec = (double*)alloc((size_t)std::max(cfg->max_iterations, 1) * 4 * sizeof(double));
    if (!dst || !dtl || !drows || !drec) return NGF_ENOMEM;
    const size_t vb = (size_t)n * sizeof(T);

    GState<T> h;
    std::memset(&h, 0, sizeof(h));
    h.cfg = {cfg->c1, cfg->step_shrink, cfg->initial_step, cfg->tol_J, cfg->tol_grad, cfg->tol_step,
             cfg->max_ls_steps, cfg->memory, cfg->max_iterations, cfg->min_iterations, max_rows};
    h.J = J;
    h.g0_inf = g0_inf;
    h.x_scale = x_scale;
    h.evals = evals0;
    h.nrows = nrows0;
    h.stop = NGF_STOP_MAX_ITER;
    const int nslots = cfg->memory + 1;
    for (int j = 0; j < nslots; ++j) {
        h.slot_s[j] = (T*)alloc(vb);
        h.slot_y[j] = (T*)alloc(vb);
        if (!h.slot_s[j] || !h.slot_y[j]) return NGF_ENOMEM;
        h.freel[h.nfree++] = nslots - 1 - j;
    }
    h.rows = drows;
    h.rec = drec;
    h.scal = scal;
    h.stats = stats;
    h.tl = dtl;
    TwoLoopArgs<T> tl;
    std::memset(&tl, 0, sizeof(tl));
    tl.gamma = 1.0;
    tl.g = g;
    tl.d = d;
    tl.n = n;
    tl.parts = parts;
    tl.slope = scal + 3;

    const auto tb0 = std::chrono::steady_clock::now();
    cudaGraph_t top = nullptr;
    cudaGraphExec_t exec = nullptr;
    Streams cs;
    struct Cleanup {
        cudaGraph_t& g;
        cudaGraphExec_t& e;
        ~Cleanup() {
            if (e) cudaGraphExecDestroy(e);
            if (g) cudaGraphDestroy(g);
        }
    } cleanup{top, exec};
    NGF_CUDA(cudaGraphCreate(&top, 0));
    NGF_CUDA(cudaGraphConditionalHandleCreate(&h.h_iter, top, 1, cudaGraphCondAssignDefault));
    NGF_CUDA(cudaGraphConditionalHandleCreate(&h.h_sd, top, 0, 0));
    NGF_CUDA(cudaGraphConditionalHandleCreate(&h.h_ls, top, 0, 0));
    NGF_CUDA(cudaGraphConditionalHandleCreate(&h.h_ok, top, 0, 0));
    NGF_CUDA(cudaGraphConditionalHandleCreate(&h.h_exp, top, 0, 0));
    for (auto& x : cs.s) NGF_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));

    cudaGraph_t body;
    {
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h.h_iter;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        NGF_CUDA(cudaGraphAddNode(&node, top, nullptr, 0, &p));
        body = p.conditional.phGraph_out[0];
    }
    const unsigned nb = blocks_for(n, 256);
    auto eval = [&](const T* y, T* gr, cudaStream_t st) { return ngf_level_eval(level, y, gr, scal, exact, st); };
    auto capture = [&](cudaGraph_t gph, cudaStream_t st, auto&& fill) -> int {
        NGF_CUDA(cudaStreamBeginCaptureToGraph(st, gph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        const int r = fill(st);
        cudaGraph_t out;
        const cudaError_t e = cudaStreamEndCapture(st, &out);
        if (r) return r;
        return (int)e;
    };
    double* t_dev = &dst->t;
    double* ttry_dev = &dst->t_try;

    // ---- the iteration body
    GRUN(capture(body, cs.s[0], [&](cudaStream_t c0) -> int {
        int rc = 0;
        NGF_LAUNCH(k_ctl_begin<T>, 1, 1, 0, c0, dst);
        GRUN(two_loop_dev_launch<T>(dtl, n, c0));
        GRUN(axpy_dev_launch<T>(x, t_dev, d, xn, n, c0));
        GRUN(eval(xn, gn, c0));
        NGF_LAUNCH(k_ctl_first<T>, 1, 1, 0, c0, dst);
        cudaGraph_t b_sd, b_ls, b_ok;
        GRUN(add_cond(c0, h.h_sd, cudaGraphCondTypeIf, &b_sd));
        GRUN(capture(b_sd, cs.s[1], [&](cudaStream_t c1) -> int {
            int rc = 0;
            GRUN(two_loop_dev_launch<T>(dtl, n, c1));
            GRUN(axpy_dev_launch<T>(x, t_dev, d, xn, n, c1));
            GRUN(eval(xn, gn, c1));
            NGF_LAUNCH(k_ctl_sd<T>, 1, 1, 0, c1, dst);
            return (int)cudaGetLastError();
        }));
        NGF_LAUNCH(k_ctl_ls_cond<T>, 1, 1, 0, c0, dst);
        GRUN(add_cond(c0, h.h_ls, cudaGraphCondTypeWhile, &b_ls));
        GRUN(capture(b_ls, cs.s[1], [&](cudaStream_t c1) -> int {
            int rc = 0;
            NGF_LAUNCH(k_ctl_shrink<T>, 1, 1, 0, c1, dst);
            GRUN(axpy_dev_launch<T>(x, t_dev, d, xn, n, c1));
            GRUN(eval(xn, gn, c1));
            NGF_LAUNCH(k_ctl_ls<T>, 1, 1, 0, c1, dst);
            return (int)cudaGetLastError();
        }));
        NGF_LAUNCH(k_ctl_post_ls<T>, 1, 1, 0, c0, dst);
        GRUN(add_cond(c0, h.h_ok, cudaGraphCondTypeIf, &b_ok));
        GRUN(capture(b_ok, cs.s[1], [&](cudaStream_t c1) -> int {
            int rc = 0;
            cudaGraph_t b_exp;
            GRUN(add_cond(c1, h.h_exp, cudaGraphCondTypeWhile, &b_exp));
            GRUN(capture(b_exp, cs.s[2], [&](cudaStream_t c2) -> int {
                int rc = 0;
                GRUN(axpy_dev_launch<T>(x, ttry_dev, d, xt, n, c2));
                GRUN(eval(xt, gt, c2));
                NGF_LAUNCH(k_ctl_exp<T>, 1, 1, 0, c2, dst);
                NGF_LAUNCH(k_copy_if<T>, nb, 256, 0, c2, dst, xt, gt, xn, gn, n);
                return (int)cudaGetLastError();
            }));
            NGF_LAUNCH(k_ctl_pair_pre<T>, 1, 1, 0, c1, dst);
            GRUN(pair_dev_launch<T>(xn, x, gn, g, &dst->cur_s, &dst->cur_y, n, stats, c1, s));
            NGF_LAUNCH(k_ctl_end<T>, 1, 1, 0, c1, dst);
            NGF_CUDA(cudaMemcpyAsync(x, xn, vb, cudaMemcpyDeviceToDevice, c1));
            NGF_CUDA(cudaMemcpyAsync(g, gn, vb, cudaMemcpyDeviceToDevice, c1));
            return (int)cudaGetLastError();
        }));
        return (int)cudaGetLastError();
    }));
    NGF_CUDA(cudaGraphInstantiate(&exec, top, 0));
    const auto tb1 = std::chrono::steady_clock::now();

    // initial state, then the whole loop in one launch
    NGF_CUDA(cudaMemcpyAsync(dst, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    NGF_CUDA(cudaMemcpyAsync(dtl, &tl, sizeof(tl), cudaMemcpyHostToDevice, s));
    if (nrows0 > 0 && max_rows > 0)
        NGF_CUDA(cudaMemcpyAsync(drows, row0, (size_t)std::min(nrows0, max_rows) * 3 * sizeof(double),
                                 cudaMemcpyHostToDevice, s));
    launched = true;
    NGF_CUDA(cudaGraphLaunch(exec, s));
    NGF_CUDA(cudaMemcpyAsync(&h, dst, sizeof(h), cudaMemcpyDeviceToHost, s));
    NGF_CUDA(cudaStreamSynchronize(s));
    if (std::getenv("NGF_GRAPH_DEBUG")) {
        const auto tb2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "graph level n=%lld: build+instantiate %.3f ms, run %.3f ms, %d iterations, %d evals\n",
                     (long long)n, std::chrono::duration<double, std::milli>(tb1 - tb0).count(),
                     std::chrono::duration<double, std::milli>(tb2 - tb1).count(), h.iter, h.evals);
    }
    res->iterations = h.iter;
    res->evaluations = h.evals;
    res->stop = h.stop;
    res->line_search_failed = h.ls_failed;
    res->rows = h.nrows;
    if (rows && max_rows > 0)
        NGF_CUDA(cudaMemcpyAsync(rows, drows, (size_t)std::min(h.nrows, max_rows) * 3 * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
    if (rec && h.iter > 0)
        NGF_CUDA(cudaMemcpyAsync(rec, drec, (size_t)h.iter * 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    NGF_CUDA(cudaStreamSynchronize(s));
    return 0;
}

template int run_level_graph<float>(ngf_level_t*, int, float*, float*, float*, float*, float*, float*, float*,
                                    double*, double*, int64_t, const ngf_lbfgs_cfg_t*, double, double, double,
                                    int, int, const double*, ngf_lbfgs_result_t*, double*, double*, int,
                                    cudaStream_t, std::vector<void*>&, bool&);
template int run_level_graph<double>(ngf_level_t*, int, double*, double*, double*, double*, double*, double*,
                                     double*, double*, double*, int64_t, const ngf_lbfgs_cfg_t*, double, double,
                                     double, int, int, const double*, ngf_lbfgs_result_t*, double*, double*,
                                     int, cudaStream_t, std::vector<void*>&, bool&);

}  // namespace ngf
