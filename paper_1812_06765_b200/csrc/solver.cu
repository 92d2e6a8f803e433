// The L-BFGS driver of one level in native code (lbfgs.py:94-181), for the device
// objective: the same decisions as the Python driver (paper_1812_06765_b200/lbfgs.py) --
// two-loop direction, steepest-descent safeguard, Armijo backtracking with forward
// expansion at t == 1, curvature-filtered history with ageing, the three relative stopping
// tests -- with the scalars it branches on read through one pinned buffer per host round
// trip.  Used by `register` for LevelObjective levels; any other callable runs the Python
// driver.

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lbfgs.cuh"

namespace ngf {

// solver_graph.cu: the iteration loop as one graph with device-side control
template <typename T>
int run_level_graph(ngf_level_t* level, int exact, T* x, T* g, T* d, T* xn, T* gn, T* xt, T* gt,
                    double* scal, double* stats, int64_t n, const ngf_lbfgs_cfg_t* cfg, double J,
                    double g0_inf, double x_scale, int evals0, int nrows0, const double* row0,
                    ngf_lbfgs_result_t* res, double* rec, double* rows, int max_rows, cudaStream_t s,
                    std::vector<void*>& owned, bool& launched);

namespace {


// The host-driven loop's scalars (J, D, S, slope at [0..3], the vector statistics at
// [8..12]) live in mapped page-locked memory: the kernels that produce them store straight
// to the host, so a round trip is one stream synchronisation with no copy behind it.
struct MappedScalars {
    double* host = nullptr;
    double* dev = nullptr;
    ~MappedScalars() {
        if (host) cudaFreeHost(host);
    }
};
thread_local MappedScalars t_map;

int mapped_scalars(double** host, double** dev) {
    if (!t_map.host) {
        if (cudaHostAlloc((void**)&t_map.host, 16 * sizeof(double), cudaHostAllocMapped) != cudaSuccess)
            return NGF_ENOMEM;
        if (cudaHostGetDevicePointer((void**)&t_map.dev, t_map.host, 0) != cudaSuccess) {
            cudaFreeHost(t_map.host);
            t_map.host = nullptr;
            return NGF_ENOMEM;
        }
    }
    *host = t_map.host;
    *dev = t_map.dev;
    return 0;
}

// scalars stored by the kernels into mapped memory: wait for the stream, then read
int read_mapped(const double* host_src, int k, double* out, cudaStream_t s) {
    NGF_CUDA(cudaStreamSynchronize(s));
    std::memcpy(out, host_src, k * sizeof(double));
    return 0;
}

// 1: run the iteration loop as one graph when eligible (NGF_LBFGS_GRAPH=1 or
// ngf_lbfgs_set_graph(1)).  Off by default: measured at 256^3 / 4 levels, the graph run of
// a level is ~1 ms faster than the host-driven loop on the 64^3 level but building and
// instantiating it costs ~0.5 ms per level, so a registration is not faster.
std::atomic<int> g_graph_mode{-1};
std::atomic<int64_t> g_graph_runs{0};
int graph_mode() {
    int m = g_graph_mode.load(std::memory_order_relaxed);
    if (m < 0) {
        const char* e = std::getenv("NGF_LBFGS_GRAPH");
        m = (e && std::atoi(e) != 0) ? 1 : 0;
        g_graph_mode.store(m, std::memory_order_relaxed);
    }
    return m;
}

struct Pair {
    void* s;
    void* y;
    double sy, yy;
};

}  // namespace
}  // namespace ngf

using namespace ngf;

extern "C" int64_t ngf_lbfgs_graph_runs(void) { return g_graph_runs.load(); }

extern "C" int ngf_lbfgs_set_graph(int on) {
    const int prev = graph_mode();
    g_graph_mode.store(on ? 1 : 0, std::memory_order_relaxed);
    return prev;
}

extern "C" int ngf_lbfgs_run_level(ngf_level_t* level, int dtype, int exact, void* x_io, int64_t n,
                                   const ngf_lbfgs_cfg_t* cfg, ngf_lbfgs_result_t* res, double* rec,
                                   double* rows, int max_rows, void* stream) {
    if (!level || !x_io || !cfg || !res || n <= 0 || (dtype != NGF_F32 && dtype != NGF_F64) ||
        cfg->memory < 1 || cfg->max_iterations < 0 || max_rows < 1)
        return NGF_EARG;
    cudaStream_t s = as_stream(stream);
    const size_t vb = (size_t)n * (dtype == NGF_F32 ? 4 : 8);
    std::memset(res, 0, sizeof(*res));

    // workspace: g, d, xn, gn, xt, gt, a copy of x, the pair pool, scalars
    std::vector<void*> owned;
    auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (dev_alloc(&p, bytes)) return nullptr;
        owned.push_back(p);
        return p;
    };
    void *x = alloc(vb), *g = alloc(vb), *d = alloc(vb), *xn = alloc(vb), *gn = alloc(vb), *xt = alloc(vb),
         *gt = alloc(vb);
    double* scal = (double*)alloc(4 * sizeof(double));   // J, D, S, slope (graph-driven loop)
    double* stats = (double*)alloc(5 * sizeof(double));  // see ngf_vec_stats / ngf_lbfgs_pair
    std::vector<Pair> free_pairs;
    int rc = (x && g && d && xn && gn && xt && gt && scal && stats) ? 0 : NGF_ENOMEM;
    double *hm = nullptr, *dm = nullptr;  // host-driven loop: mapped scalars
    if (!rc) rc = mapped_scalars(&hm, &dm);
    double* const mscal = dm;      // J, D, S, slope
    double* const mstats = dm + 8;  // vector statistics
    auto cleanup = [&]() {
        cudaStreamSynchronize(s);
        for (void* p : owned) dev_free(p);
    };
    if (rc) {
        cleanup();
        return rc;
    }
    cudaMemcpyAsync(x, x_io, vb, cudaMemcpyDeviceToDevice, s);

    int nrows = 0;
    auto row = [&](const double* v) {
        if (nrows < max_rows) {
            rows[3 * nrows] = v[0];
            rows[3 * nrows + 1] = v[1];
            rows[3 * nrows + 2] = v[2];
        }
        ++nrows;
    };
    double sc[5];
#define RUN(call)               \
    do {                        \
        rc = (call);            \
        if (rc) goto done;      \
    } while (0)

    {
        int evals = 0;
        RUN(ngf_level_eval(level, x, g, mscal, exact, s));
        ++evals;
        RUN(read_mapped(hm, 3, sc, s));
        double J = sc[0];
        row(sc);
        RUN(ngf_vec_stats(dtype, g, nullptr, x, nullptr, n, mstats, s));
        double st[5];
        RUN(read_mapped(hm + 8, 5, st, s));
        const double g0_inf = st[4];
        if (g0_inf <= 0.0) {
            res->stop = NGF_STOP_STATIONARY;  // (the reference reports no evaluations here)
            goto done;
        }
        if (cfg->max_iterations > 0 && cfg->max_ls_steps < 1) {
            // no trial step may be evaluated: the reference's backtracking loop runs zero
            // times and reports a failed line search (lbfgs.py:121-132)
            res->stop = NGF_STOP_LINE_SEARCH;
            res->line_search_failed = 1;
            res->evaluations = evals;
            goto done;
        }
        std::vector<Pair> history;
        const double x_scale = std::max(std::sqrt(st[2]), 1.0);
        // the whole loop as one graph launch when the two-loop fits the cluster kernel
        // (NGF_LBFGS_GRAPH=0 keeps the host-driven loop below)
        if (graph_mode() && cfg->max_iterations > 0 && n <= kTwoLoopClusterMaxN) {
            bool launched = false;
            const double row0[3] = {sc[0], sc[1], sc[2]};
            rc = dtype == NGF_F32
                     ? run_level_graph<float>(level, exact, (float*)x, (float*)g, (float*)d, (float*)xn,
                                              (float*)gn, (float*)xt, (float*)gt, scal, stats, n, cfg, J,
                                              g0_inf, x_scale, evals, nrows, row0, res, rec, rows, max_rows, s,
                                              owned, launched)
                     : run_level_graph<double>(level, exact, (double*)x, (double*)g, (double*)d, (double*)xn,
                                               (double*)gn, (double*)xt, (double*)gt, scal, stats, n, cfg, J,
                                               g0_inf, x_scale, evals, nrows, row0, res, rec, rows, max_rows,
                                               s, owned, launched);
            if (!rc) {
                nrows = res->rows;
                g_graph_runs.fetch_add(1, std::memory_order_relaxed);
                goto done;
            }
            if (launched) goto done;
            cudaGetLastError();  // graph construction failed before launch: host-driven loop
            rc = 0;
        }
        int rejected = 0;
        auto two_loop = [&]() {
            const int m = (int)history.size();
            std::vector<const void*> S(std::max(m, 1)), Y(std::max(m, 1));
            std::vector<double> rho(std::max(m, 1));
            for (int k = 0; k < m; ++k) {
                S[k] = history[k].s;
                Y[k] = history[k].y;
                rho[k] = 1.0 / history[k].sy;
            }
            const double gamma = m ? history[m - 1].sy / history[m - 1].yy : 1.0;
            return ngf_lbfgs_two_loop(dtype, S.data(), Y.data(), rho.data(), gamma, m, g, d, n, mscal + 3, s);
        };
        // Speculation on small levels (an evaluation costs about as much as a host round
        // trip there): the first forward-expansion trial (t = 2 t0 into xt / gt, its scalars
        // in slots 4..6) is issued together with the first trial when the previous
        // iteration accepted its first trial, and used only if the reference's control flow
        // reaches it (Armijo holds at t0, no safeguard); otherwise it is dropped uncounted.
        // The evaluations, their order and every decision are those of the serial loop.
        static const bool spec_on = !(std::getenv("NGF_LBFGS_SPEC") && std::atoi(std::getenv("NGF_LBFGS_SPEC")) == 0);
        const bool spec_level = spec_on && n <= 3 * 32768 && cfg->max_ls_steps > 1;
        bool t0_accepted = true;
        for (int it = 0; it < cfg->max_iterations; ++it) {
            // direction and (optimistically) the first trial point, one host round trip
            RUN(two_loop());
            double t = cfg->initial_step;
            RUN(ngf_vec_axpy_step(dtype, x, t, d, xn, n, s));
            RUN(ngf_level_eval(level, xn, gn, mscal, exact, s));
            ++evals;
            bool have_spec = spec_level && t0_accepted;
            if (have_spec) {
                RUN(ngf_vec_axpy_step(dtype, x, t / cfg->step_shrink, d, xt, n, s));
                RUN(ngf_level_eval(level, xt, gt, mscal + 4, exact, s));
            }
            double v[4];
            RUN(read_mapped(hm, 4, v, s));
            double Jn = v[0], slope = v[3];
            int ls_evals = 1;
            if (slope >= 0) {  // safeguard: steepest descent (lbfgs.py:113-116)
                have_spec = false;
                --evals;       // the optimistic trial above is discarded
                for (const Pair& p : history) free_pairs.push_back(p);
                history.clear();
                RUN(two_loop());
                RUN(ngf_vec_axpy_step(dtype, x, t, d, xn, n, s));
                RUN(ngf_level_eval(level, xn, gn, mscal, exact, s));
                ++evals;
                RUN(read_mapped(hm, 4, v, s));
                Jn = v[0];
                slope = v[3];
            }
            row(v);
            bool accepted = false;
            while (true) {
                if (std::isfinite(Jn) && Jn <= J + cfg->c1 * t * slope) {
                    accepted = true;
                    break;
                }
                have_spec = false;
                if (ls_evals >= cfg->max_ls_steps) break;
                t *= cfg->step_shrink;
                RUN(ngf_vec_axpy_step(dtype, x, t, d, xn, n, s));
                RUN(ngf_level_eval(level, xn, gn, mscal, exact, s));
                ++evals;
                RUN(read_mapped(hm, 3, v, s));
                Jn = v[0];
                row(v);
                ++ls_evals;
            }
            if (!accepted) {
                res->stop = NGF_STOP_LINE_SEARCH;
                res->line_search_failed = 1;
                res->evaluations = evals;
                goto done;
            }
            t0_accepted = t == cfg->initial_step;
            if (t == cfg->initial_step) {
                // forward expansion while Armijo holds and J decreases (lbfgs.py:133-143)
                while (ls_evals < cfg->max_ls_steps) {
                    const double t_try = t / cfg->step_shrink;
                    if (have_spec) {  // already evaluated, issued with the first trial
                        have_spec = false;
                        std::memcpy(v, hm + 4, 3 * sizeof(double));
                    } else {
                        RUN(ngf_vec_axpy_step(dtype, x, t_try, d, xt, n, s));
                        RUN(ngf_level_eval(level, xt, gt, mscal, exact, s));
                        RUN(read_mapped(hm, 3, v, s));
                    }
                    ++evals;
                    const double Jt = v[0];
                    row(v);
                    ++ls_evals;
                    if (std::isfinite(Jt) && Jt <= J + cfg->c1 * t_try * slope && Jt < Jn) {
                        t = t_try;
                        Jn = Jt;
                        std::swap(xn, xt);
                        std::swap(gn, gt);
                    } else {
                        break;
                    }
                }
            }
            // history pair and stopping statistics in one pass (lbfgs.py:145-164)
            Pair pair;
            if (!free_pairs.empty()) {
                pair = free_pairs.back();
                free_pairs.pop_back();
            } else {
                pair.s = alloc(vb);
                pair.y = alloc(vb);
                if (!pair.s || !pair.y) {
                    rc = NGF_ENOMEM;
                    goto done;
                }
            }
            RUN(ngf_lbfgs_pair(dtype, xn, x, gn, g, pair.s, pair.y, n, mstats, s));
            RUN(read_mapped(hm + 8, 4, st, s));
            const double sy = st[0], ss = st[1], yy = st[2], g_inf = st[3];
            pair.sy = sy;
            pair.yy = yy;
            if (sy > 1e-10 * std::sqrt(ss) * std::sqrt(yy)) {
                history.push_back(pair);
                if ((int)history.size() > cfg->memory) {
                    free_pairs.push_back(history.front());
                    history.erase(history.begin());
                }
                rejected = 0;
            } else {
                free_pairs.push_back(pair);
                ++rejected;
                if (!history.empty()) {
                    free_pairs.push_back(history.front());
                    history.erase(history.begin());
                }
                if (rejected >= cfg->memory) {
                    for (const Pair& p : history) free_pairs.push_back(p);
                    history.clear();
                }
            }
            const double step_norm = std::sqrt(ss);
            const double J_prev = J;
            std::swap(x, xn);
            std::swap(g, gn);
            J = Jn;
            if (rec) {
                rec[4 * it] = J;
                rec[4 * it + 1] = g_inf;
                rec[4 * it + 2] = t;
                rec[4 * it + 3] = ls_evals;
            }
            res->iterations = it + 1;
            if (it + 1 >= cfg->min_iterations) {
                if (std::fabs(J_prev - J) <= cfg->tol_J * std::max(std::fabs(J_prev), 1e-30)) {
                    res->stop = NGF_STOP_OBJECTIVE;
                    break;
                }
                if (g_inf <= cfg->tol_grad * g0_inf) {
                    res->stop = NGF_STOP_GRADIENT;
                    break;
                }
                if (step_norm <= cfg->tol_step * x_scale) {
                    res->stop = NGF_STOP_STEP;
                    break;
                }
            }
            if (it + 1 == cfg->max_iterations) res->stop = NGF_STOP_MAX_ITER;
        }
        if (cfg->max_iterations == 0) res->stop = NGF_STOP_MAX_ITER;
        res->evaluations = evals;
    }
done:
#undef RUN
    res->rows = nrows;
    if (!rc) cudaMemcpyAsync(x_io, x, vb, cudaMemcpyDeviceToDevice, s);  // the final (accepted) x
    cleanup();
    return rc;
}
