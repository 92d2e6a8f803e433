/*
 * ngf_b200.h -- C-ABI of libngfb200.so, the B200 (sm_100a) implementation of the
 * matrix-free NGF + curvature objective/gradient hot path of arXiv 1812.06765.
 *
 * The reference (`ngfreg`, /root/reference/pkg/src/ngfreg) is pure Python with
 * no FFI; every entry point below names the reference function it replaces.
 * INTEGRATION.md shows the ctypes stubs a maintainer adds to the reference.
 *
 * Conventions (reference geometry.py:1-10, objective.py:1-6):
 *   - volumes are C-order (nz, ny, nx), x fastest; vector fields (3, nz, ny, nx)
 *     with components (x, y, z); the flat optimisation variable is their ravel;
 *   - all array pointers are DEVICE pointers owned by the caller, unless the
 *     parameter name says `host_`; the library never frees caller memory;
 *   - `dtype` is NGF_F32 or NGF_F64 (the reference's `precision`, geometry.py:170-181);
 *   - every call is stream-ordered on `stream` (a cudaStream_t, 0 = legacy default);
 *   - return value: 0 ok; > 0 a cudaError_t; < 0 one of the NGF_E* argument errors.
 *     Grid mismatches return NGF_EGRID (the host wrapper raises GridError, as the
 *     reference does in transfer.py:42-51).
 */
#ifndef NGF_B200_H
#define NGF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGF_F32 0
#define NGF_F64 1

#define NGF_OK 0
#define NGF_EARG (-1)     /* bad argument (null pointer, bad dtype, bad size)        */
#define NGF_EGRID (-2)    /* grids do not cover the same domain / dims incompatible   */
#define NGF_ENOMEM (-3)   /* device or host allocation failed                        */
#define NGF_ESTATE (-4)   /* handle used in the wrong state                          */

/* Cell-centred axis-aligned grid (reference Grid3, geometry.py:24-43):
 * dims = (nx, ny, nz), spacing in mm, origin = world position of cell (0,0,0). */
typedef struct ngf_grid {
    int64_t dims[3];
    double spacing[3];
    double origin[3];
} ngf_grid_t;

typedef struct ngf_plan ngf_plan_t;    /* grid-transfer plan (def grid -> image grid) */
typedef struct ngf_level ngf_level_t;  /* one multilevel level: template, reference terms, workspace */

int ngf_version(void);
/* Number of CUDA kernel launches issued by this library since load (for bench.py's gpu_launches). */
int64_t ngf_launch_count(void);
const char* ngf_error_string(int code);

/* ---------------------------------------------------------------- plans (host, f64, bit-exact)
 * Replaces transfer.py:54-63 (_axis_transfer), :82-110 (build_gather_plan) and the
 * compatibility check transfer.py:42-51.  The plan is computed on the host in IEEE
 * double with no contraction, then uploaded (f32 and f64 copies of the weights).   */
int ngf_plan_create(const ngf_grid_t* def_grid, const ngf_grid_t* img_grid, ngf_plan_t** out);
/* prolongation plan (multilevel.py:163-176): like ngf_plan_create but only checks
 * that the grids cover the same domain (no dims ordering requirement). */
int ngf_plan_create_prolong(const ngf_grid_t* coarse, const ngf_grid_t* fine, ngf_plan_t** out);
void ngf_plan_destroy(ngf_plan_t* plan);
/* Copy one axis of the plan to host arrays (sizes: i0/w1 n_img, start/counts n_def,
 * weights n_def*width).  Pass NULL arrays to only query width. */
int ngf_plan_axis(const ngf_plan_t* plan, int axis, int32_t* host_i0, double* host_w1,
                  int32_t* host_start, int32_t* host_counts, double* host_weights, int32_t* width);

/* ---------------------------------------------------------------- standalone operators
 * Bit-exact re-statements of the reference operators (same IEEE operation order).  */

/* yhat = P y (transfer.py:129-148); y (3, def), yhat (3, img). */
int ngf_apply_P(const ngf_plan_t* plan, int dtype, const void* y, void* yhat, void* stream);
/* out = P^T r, deterministic gather (transfer.py:173-192, the "gather" variant). */
int ngf_apply_Pt(const ngf_plan_t* plan, int dtype, const void* r, void* out, void* stream);
/* out = P^T r with the reference's variant `variant`: NGF_PT_GATHER (= ngf_apply_Pt),
 * NGF_PT_SCATTER (transfer.py:199-222, float atomics: equal to the gather up to
 * reassociation), NGF_PT_REDBLACK (transfer.py:225-256, two parity launches:
 * bit-identical to the reference's red-black). */
#define NGF_PT_GATHER 0
#define NGF_PT_SCATTER 1
#define NGF_PT_REDBLACK 2
int ngf_apply_Pt_variant(const ngf_plan_t* plan, int dtype, int variant, const void* r, void* out,
                         void* stream);
/* out(n,3) = trilinear value of the deformation y (3, grid) at the world points
 * pts(n,3), clamp-to-edge, in f64 (evaluation.py:39-64 `sample_deformation`; landmark
 * and probe evaluation). */
int ngf_sample_field(const ngf_grid_t* grid, int dtype, const void* y, const double* pts, int64_t n,
                     double* out, void* stream);
/* W = T(yhat), mask (warp.py:64-90).  mask may be NULL. */
int ngf_warp(const ngf_grid_t* tgrid, int dtype, const void* T, const void* yhat, int64_t n,
             void* W, uint8_t* mask, void* stream);
/* out(3,n) = s * grad T~(yhat) / h, zero outside the hull (warp.py:93-127). */
int ngf_warp_jt(const ngf_grid_t* tgrid, int dtype, const void* T, const void* yhat,
                const void* s, int64_t n, void* out, void* stream);
/* G and G^T on one grid (warp.py:130-184). */
int ngf_gradient(const ngf_grid_t* grid, int dtype, const void* v, void* out3, void* stream);
int ngf_gradient_t(const ngf_grid_t* grid, int dtype, const void* w3, void* out, void* stream);
/* grad R and ||grad R||_rho (ngf.py:60-67). */
int ngf_ref_terms(const ngf_grid_t* grid, int dtype, const void* R, double rho, void* gR3,
                  void* nR, void* stream);
/* Per voxel terms 1 - r^2 and q (ngf.py:70-80, :93-112), W given. */
int ngf_ngf_terms(const ngf_grid_t* grid, int dtype, const void* W, const void* gR3,
                  const void* nR, double tau, double rho, void* terms, void* q3, void* stream);
/* numpy-pairwise sum of n values (the np.sum of ngf.py:90 / curvature.py:70), written as
 * a double to *out_dev (the exact working-dtype value). */
int ngf_pairwise_sum(int dtype, const void* x, int64_t n, double* out_dev, void* stream);
/* 7-point Laplacian with zero face rows and its transpose (curvature.py:20-45), one component. */
int ngf_laplacian(const ngf_grid_t* grid, int dtype, const void* u, void* out, void* stream);
int ngf_laplacian_t(const ngf_grid_t* grid, int dtype, const void* w, void* out, void* stream);
/* S and grad S = vol L^T L (y - id) (curvature.py:63-81).  S written to *S_dev. */
int ngf_curvature(const ngf_grid_t* grid, int dtype, const void* y, double* S_dev, void* grad,
                  void* stream);
/* 2x2x2 block mean, axes z, y, x in turn (multilevel.py:100-121); out dims ceil(n/2). */
int ngf_downsample(const ngf_grid_t* in_grid, int dtype, const void* in, void* out, void* stream);
/* y_fine = id_fine + P_(coarse->fine)(y - id_coarse) (multilevel.py:163-176). */
int ngf_prolong(const ngf_plan_t* prolong_plan, int dtype, const void* y_coarse, void* y_fine,
                void* stream);

/* ---------------------------------------------------------------- level objective
 * Replaces LevelObjective (objective.py:22-60) + distance_and_gradient (ngf.py:117-134)
 * + precompute_reference_terms (ngf.py:60-67).  T and R are device volumes on
 * img_grid; T must stay alive for the life of the level (it is read, not copied).  */
int ngf_level_create(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                     const void* T, const void* R, double tau, double rho, double alpha,
                     void* stream, ngf_level_t** out);
/* Same, from precomputed reference terms gR (3, N) and nR (N) (the reference's
 * LevelObjective receives ReferenceTerms, objective.py:27); both are copied. */
int ngf_level_create_terms(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                           const void* T, const void* gR, const void* nR, double tau, double rho,
                           double alpha, void* stream, ngf_level_t** out);
void ngf_level_destroy(ngf_level_t* level);
/* One objective+gradient evaluation: grad (3M) = grad D + alpha grad S, and
 * scalars_dev[0..2] = (J, D, S) as doubles with the reference's rounding.
 * mode 0 = fused sm_100a kernels (performance path),
 * mode 1 = exact path (reference operation order, bit-exact D and grad D). */
int ngf_level_eval(ngf_level_t* level, const void* y, void* grad, double* scalars_dev, int mode,
                   void* stream);
/* The same evaluation with host arrays, synchronous: y_host (3M values, pageable or
 * page-locked) is uploaded through the library's staging threads, grad_host receives the
 * gradient and scalars_host[0..2] = (J, D, S).  mode 0 or 1 as above.  This is the
 * reference's LevelObjective.__call__(x) -> (J, grad) (objective.py:48-60) for callers
 * that hold numpy / host memory. */
int ngf_level_eval_host(ngf_level_t* level, const void* y_host, void* grad_host,
                        double* scalars_host, int mode, void* stream);
/* Pipelining of ngf_level_eval_host (mode 0, lean march, both host arrays page-locked):
 * the level's z chunks run as `parts` groups on their own streams, each group starting
 * once its deformation planes are uploaded, and the planes a group finalises go down
 * while later groups march.  Results are bit-identical to the serial call.  parts 0 =
 * the default (4, or NGF_PIPE_PARTS), 1 = serial, at most 8. */
int ngf_level_set_host_pipeline(ngf_level_t* level, int parts);
/* Host <-> device copies staged through page-locked memory by the library's copy threads
 * (a pageable cudaMemcpy runs at a fraction of the PCIe bandwidth).  ngf_host_upload is
 * stream-ordered; a pageable src_host may be reused when it returns, a page-locked one is
 * copied by a direct asynchronous DMA and must stay unchanged until the stream has passed
 * the copy (cudaMemcpyAsync semantics).  ngf_host_download returns once dst_host holds
 * the data (it synchronises the stream). */
int ngf_host_upload(void* dst_dev, const void* src_host, size_t bytes, void* stream);
int ngf_host_download(void* dst_host, const void* src_dev, size_t bytes, void* stream);
/* 1 when host_ptr lies in page-locked (cudaHostAlloc / registered) memory, else 0: the
 * Python layer keeps such upload sources alive until their asynchronous DMA completed. */
int ngf_host_is_pinned(const void* host_ptr);
/* Config-5 z-slab decomposition: restrict the fused evaluation to image
 * planes [zlo, zhi).  mode 2 of ngf_level_eval then writes the slab's NGF partial
 * (grad <- grad D_slab, scalars[1] <- D_slab, no curvature); after summing grad and
 * scalars[1] over slabs (e.g. an NCCL all-reduce), ngf_level_add_curvature adds
 * alpha grad S and sets scalars = (J, D, S), identically on every rank. */
/* A config-5 slab level: like ngf_level_create, but the reference terms are computed on
 * image planes [zlo, zhi) only (R itself is read on the neighbouring planes, so no halo
 * exchange is needed) and the fused march is restricted to that slab.  Only mode 2 of
 * ngf_level_eval and ngf_level_add_curvature are valid on it (NGF_ESTATE otherwise). */
int ngf_level_create_zslab(const ngf_grid_t* img_grid, const ngf_grid_t* def_grid, int dtype,
                           const void* T, const void* R, double tau, double rho, double alpha,
                           int64_t zlo, int64_t zhi, void* stream, ngf_level_t** out);
int ngf_level_set_zrange(ngf_level_t* level, int64_t zlo, int64_t zhi);
int ngf_level_add_curvature(ngf_level_t* level, const void* y, void* grad, double* scalars_dev,
                            void* stream);
/* Device pointer of the level's reference terms (packed (gx, gy, gz, 1) / nR per voxel). */
const void* ngf_level_ref_terms(const ngf_level_t* level);
/* P^T variant used by the exact evaluation (mode 1): NGF_PT_GATHER (default),
 * NGF_PT_SCATTER or NGF_PT_REDBLACK (objective.py:22-60 `pt_variant`).  The fused
 * evaluation always uses its deterministic tile gather. */
int ngf_level_set_pt_variant(ngf_level_t* level, int variant);
/* Record CUDA events around the fused kernel of every mode-0 evaluation (bench.py's
 * roofline), and read the last one's duration in ms (synchronises on the event). */
int ngf_level_set_timing(ngf_level_t* level, int on);
int ngf_level_kernel_ms(ngf_level_t* level, float* ms);
/* info[0..8]: fused CTAs, smem bytes, z chunk, P^T window wx, wy, wz, tiles ntx, nty, ntz. */
int ngf_level_info(const ngf_level_t* level, int64_t* info);
/* Kernel variant of the level's fused march: 0-5 the classic two-slot / one-slot tile
 * shapes (fused_march.cuh), 6 the lean march (march_lean.cu; f32, power-of-two spacing,
 * grid ratio >= 2).  NGF_FUSED_VARIANT=<v> forces one when eligible, NGF_NO_LEAN=1 keeps
 * the classic ones. */
int ngf_level_variant(const ngf_level_t* level);

/* ---------------------------------------------------------------- L-BFGS vector algebra
 * lbfgs.py:68-181.  Scalars that the reference keeps as Python floats live in
 * double device memory so no host round trip is needed inside the two-loop.     */
/* out_dev[0] = sum a*b in double, deterministic order. */
int ngf_vec_dot(int dtype, const void* a, const void* b, int64_t n, double* out_dev, void* stream);
/* Batched stats in one pass: out_dev[0]=g.d, [1]=s.y, [2]=|s|^2, [3]=|y|^2, [4]=max|g|.
 * Any of s/y may be NULL (their entries are then 0). */
int ngf_vec_stats(int dtype, const void* g, const void* d, const void* s, const void* y,
                  int64_t n, double* out_dev, void* stream);
/* out = x + dtype(t) * d  (lbfgs.py:122, :137); t read from host. */
int ngf_vec_axpy_step(int dtype, const void* x, double t, const void* d, void* out, int64_t n,
                      void* stream);
/* out = a - b (lbfgs.py:145-146). */
int ngf_vec_sub(int dtype, const void* a, const void* b, void* out, int64_t n, void* stream);
/* s = x_new - x, y = g_new - g and out_dev[0..3] = (s.y, s.s, y.y, max|g_new|) in one pass
 * (lbfgs.py:145-148, :161-164). */
int ngf_lbfgs_pair(int dtype, const void* x_new, const void* x, const void* g_new, const void* g,
                   void* s_out, void* y_out, int64_t n, double* out_dev, void* stream);
/* d = -H g by the two-loop recursion over m (s, y) pairs ordered oldest first
 * (lbfgs.py:68-91), one cooperative launch.  S and Y are host arrays of m device
 * pointers; host_rho[k] = 1 / (y_k . s_k); gamma = (s.y)/(y.y) of the newest pair.
 * Writes the slope g.d to *slope_dev.  m == 0 gives d = -g. */
int ngf_lbfgs_two_loop(int dtype, const void* const* S, const void* const* Y, const double* host_rho,
                       double gamma, int m, const void* g, void* d, int64_t n, double* slope_dev,
                       void* stream);

/* ---------------------------------------------------------------- native L-BFGS driver
 * lbfgs_minimize (lbfgs.py:94-181) for a level's device objective: the reference's
 * decisions (two-loop direction, steepest-descent safeguard, Armijo backtracking with
 * forward expansion at t == 1, curvature-filtered history with ageing, relative stopping
 * tests after min_iterations) with one pinned host round trip per scalar read.          */
typedef struct {
    int memory, max_iterations, max_ls_steps, min_iterations;
    double c1, initial_step, step_shrink;       /* LbfgsConfig */
    double tol_J, tol_grad, tol_step;           /* StoppingRules */
} ngf_lbfgs_cfg_t;
#define NGF_STOP_OBJECTIVE 0
#define NGF_STOP_GRADIENT 1
#define NGF_STOP_STEP 2
#define NGF_STOP_MAX_ITER 3
#define NGF_STOP_LINE_SEARCH 4
#define NGF_STOP_STATIONARY 5
typedef struct {
    int iterations, evaluations, stop, line_search_failed, rows;
} ngf_lbfgs_result_t;
/* Minimise the level objective from the device vector x (n values of dtype, updated in
 * place with the final iterate); exact selects the bit-exact evaluation.  rec[4 * it] =
 * (J, max|g|, step, line-search evaluations) per iteration (room for max_iterations);
 * rows[3 * k] = (J, D, S) per evaluation, up to max_rows (res->rows counts them all). */
int ngf_lbfgs_run_level(ngf_level_t* level, int dtype, int exact, void* x, int64_t n,
                        const ngf_lbfgs_cfg_t* cfg, ngf_lbfgs_result_t* res, double* rec, double* rows,
                        int max_rows, void* stream);
/* Levels whose vectors fit the cluster two-loop (n <= 131072: deformation grids up to
 * ~35^3) can run the whole iteration loop as ONE CUDA graph with device-side control
 * (conditional nodes; csrc/solver_graph.cu) -- the same decisions, no host round trips --
 * when ngf_lbfgs_set_graph(1) (or NGF_LBFGS_GRAPH=1) selects it; the default is the
 * host-driven loop.  Returns the previous setting. */
int ngf_lbfgs_set_graph(int on);
/* Number of level loops that ran as a graph in this process (tests, bench). */
int64_t ngf_lbfgs_graph_runs(void);

#ifdef __cplusplus
}
#endif
#endif /* NGF_B200_H */
