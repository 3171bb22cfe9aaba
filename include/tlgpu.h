/*
 * tlgpu.h — C ABI of the B200 two-level heat-solve library (libtlgpu.so).
 *
 * The reference (lpbfsim, pure Python) has no FFI; its seams are Python
 * functions.  Each entry point below names the reference function whose work
 * it replaces; the Python host layer (paper_2110_12932_b200/) keeps the
 * reference signatures and calls these through ctypes.
 *
 * Conventions
 *   - Plain C types only; all arrays are contiguous fp64 in the reference node
 *     order  id = i + (nx+1)*(j + (ny+1)*k)  (lpbfsim/mesh.py:406-409).
 *   - Host pointers are borrowed for the duration of the call.
 *   - Every function returns TL_OK (0) or a negative TL_E* code; the message is
 *     available from tl_last_error() (thread-local).  No C++ exception crosses
 *     the ABI.  Solver non-convergence is NOT an error code: it is reported
 *     per solve in tl_solve_info.status, and the Python layer raises the
 *     reference's NonConvergence / SolverError from it.
 *   - One CUDA stream per tl_run; handles are not thread-safe, distinct handles
 *     may be used concurrently from different threads / devices.
 */
#ifndef TLGPU_H
#define TLGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLGPU_ABI_VERSION 1

enum {
    TL_OK = 0,
    TL_E_INVALID = -1,   /* bad argument                         */
    TL_E_CUDA = -2,      /* CUDA runtime failure                 */
    TL_E_NODEVICE = -3,  /* no usable sm_100 device              */
    TL_E_ALLOC = -4      /* device allocation failed             */
};

/* Dirichlet node sets the device kernels represent (structured, implicit). */
enum {
    TL_DIRICHLET_BOTTOM = 0,  /* z = lo face: global level, lpbfsim/twolevel.py:115-122     */
    TL_DIRICHLET_GAMMA = 1    /* lateral + bottom faces: local level, twolevel.py:124-131,
                                 mesh.py:498,507 (trace nodes)                              */
};

/* Per-solve outcome (mirrors what fem.solve_linear checks, fem.py:271-291). */
enum {
    TL_SOLVE_OK = 0,
    TL_SOLVE_MAXITER = 1,     /* scipy cg info != 0                     */
    TL_SOLVE_RESIDUAL = 2,    /* ||A x - b|| / ||b|| > 100 rtol         */
    TL_SOLVE_NONFINITE = 3    /* FieldState finite check, fem.py:50-51  */
};

typedef struct {
    int32_t iterations;   /* CG iterations (scipy callback count)        */
    int32_t status;       /* TL_SOLVE_*                                   */
    double bnorm;         /* ||b||_2 of the constrained system            */
    double rnorm;         /* ||r||_2 of the recursive residual at exit    */
    double true_resid;    /* ||A_c x - b||_2 / ||b||_2                    */
} tl_solve_info;

/* Structured grid: construction box, cell counts, accumulated translation. */
typedef struct {
    int32_t ncells[3];
    double lo0[3];
    double hi0[3];
    double offset[3];      /* Mesh._offset (mesh.py:164,372)              */
} tl_grid_desc;

/* Volumetric conical Gaussian (sources.py:67-77): peak = 6 sqrt3 P eta / (2 pi r^2 d). */
typedef struct {
    double peak;
    double radius;
    double depth;
    double center[3];
    int32_t on;            /* 0: no source (laser off / after path end)   */
} tl_gaussian;

/* Temperature-dependent material (materials.py:40-134): tables in K, piecewise linear
 * and clamped (np.interp); latent != 0 adds the secant apparent capacity (fem.py:197-211). */
typedef struct {
    const double* k_T;
    const double* k_v;
    int32_t nk;
    const double* c_T;
    const double* c_v;
    int32_t nc;
    double rho, chi, S, T_melt;
    int32_t latent;
} tl_vc_material;

/* Top-face Robin terms (fem.py:241-268): h_conv, sigma*emissivity (lagged T^3), T_ambient. */
typedef struct {
    double h_conv;
    double sigma_eps;
    double T_ambient;
    int32_t on;
} tl_robin;

/* Whole two-level run: both grids, constant material, BCs, solver settings. */
typedef struct {
    tl_grid_desc global_grid;
    tl_grid_desc local_grid;        /* initial placement                   */
    double kappa;                   /* W/(m K), both levels (one-way coupling) */
    double rho_c_global;            /* rho * c of the global material, J/(m^3 K) */
    double rho_c_local;             /* rho * c of the local material         */
    double T_buildplate;            /* global Dirichlet value              */
    double beam_peak, beam_radius, beam_depth;
    double rtol;                    /* SolverSettings.linear_tol           */
    int32_t maxiter_factor;         /* maxiter = factor * n  (fem.py:285: 20) */
    int32_t max_micro;              /* largest micro count per macro step  */
    int32_t max_deposit;            /* largest deposit sample count per step */
    int32_t device;                 /* CUDA device ordinal                 */
    int32_t external_planes;        /* 0: the run owns the global level.  > 0: multi-GPU
                                       local-only run — the global field comes from the
                                       z-slab solve (tl_run_put_global_planes) and only its
                                       top external_planes planes (the local box's P1
                                       support) are stored; no global solver workspace */
} tl_run_desc;

/* One macro step of the one-way multirate cycle (multirate.py:105-164), or one
 * uniform step of run_space (n_micro == 1, multirate.py:203-216).  All values are
 * precomputed on the host from the path and schedule only. */
typedef struct {
    double dt_global;               /* global step (fem.py:307, dt)        */
    int32_t dep_offset;             /* first deposit sample of this step   */
    int32_t dep_count;              /* deposit samples (SweptTrackDeposit) */
    int32_t micro_offset;           /* first tl_micro_plan of this step    */
    int32_t n_micro;                /* local solves that advance time      */
    int32_t corrector;              /* 1: re-solve the last micro interval (multirate.py:149) */
    int32_t relocate;               /* 1: local box moves after this step  */
    int32_t record;                 /* 0: no snapshots; 1: keep the predictor + every micro field;
                                       > 1 (bit 0 set): snapshot decimation (runner.py:216-233) -
                                       micro field i is kept only if bit i + 1 is set (i >= 30:
                                       always); the predictor and the step's final local field
                                       are kept whenever record != 0 */
    double new_offset[3];           /* local offset after the move          */
} tl_macro_plan;

typedef struct {
    double dt;                      /* local step length                    */
    double w;                       /* trace blend weight (multirate.py:92-102) */
    double center[3];               /* Gaussian centre at t1                */
    int32_t source_on;
} tl_micro_plan;

typedef struct tl_run tl_run;

/* ---- library ---------------------------------------------------------------- */
int32_t tl_abi_version(void);
const char* tl_last_error(void);
/* SM count, L2 bytes, cooperative-launch support of a device. */
int32_t tl_device_query(int32_t device, int32_t* sm_count, int64_t* l2_bytes, int32_t* coop);

/* ---- single implicit step: replaces fem.step_backward_euler for a linear
 *      problem (fem.py:307-355) = assemble_system (fem.py:129-194) +
 *      constrained (fem.py:89-105) + solve_linear cg (fem.py:271-291).
 *      dirichlet values: g = (1-w)*gA + w*gB on the Dirichlet set, or the
 *      constant g_const when gA == NULL.  load (dense, optional) is the
 *      extra_load / deposit term.  Host buffers in and out. */
int32_t tl_step_host(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                     int32_t dirichlet_kind, const double* gA, const double* gB, double w,
                     double g_const, const double* T_old, const double* load,
                     const tl_gaussian* src, double rtol, int32_t maxiter,
                     double* x_out, tl_solve_info* info);

/* tl_step_host with the Dirichlet data as a node list (ids and values, scattered into the
 * dense array on the device; g_const and the blend do not apply). */
int32_t tl_step_nodes_host(const tl_grid_desc* grid, double kappa, double rho_c, double dt,
                           int32_t dirichlet_kind, const int32_t* dirichlet_nodes, int64_t n_dirichlet,
                           const double* dirichlet_values, const double* T_old, const double* load,
                           const tl_gaussian* src, double rtol, int32_t maxiter, double* x_out,
                           tl_solve_info* info);

/* Device time (CUDA events) of the last tl_step_host's solve launches (RHS, CG loop,
 * residual, finish), for benchmarks and solver tuning. */
int32_t tl_step_last_ms(float* ms);

/* ---- P1 interpolation of a global field at the nodes of a (translated) grid:
 *      Mesh.interpolate (mesh.py:358-361) on Mesh.locate (mesh.py:308-339).
 *      gamma_only != 0 evaluates only the gamma nodes (InterfaceGamma.trace_of,
 *      mesh.py:471-474) and leaves the others untouched. */
int32_t tl_interpolate_host(const tl_grid_desc* global_grid, const double* values,
                            const tl_grid_desc* target, int32_t gamma_only, double* out);

/* ---- P1 interpolation at arbitrary points (Mesh.interpolate). */
int32_t tl_interpolate_points_host(const tl_grid_desc* global_grid, const double* values,
                                   const double* points, int64_t npoints, double* out);

/* ---- one Picard pass of fem.step_backward_euler for a NONLINEAR problem (fem.py:307-355):
 *      assemble_system with coefficients frozen at T_lag (fem.py:129-194: temperature-
 *      dependent kappa / c tables, latent secant capacity, lumped convection + lagged
 *      radiation on the top face, Gaussian source, extra_load), constrained (fem.py:89-105,
 *      Dirichlet set given as a node mask with values g), Jacobi-PCG with scipy's
 *      recurrences (fem.py:271-298).  x_out has x_D = g.  The caller runs the Picard loop. */
int32_t tl_vc_step_host(const tl_grid_desc* grid, const tl_vc_material* mat, double dt, const double* T_old,
                        const double* T_lag, const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                        const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, double* x_out,
                        tl_solve_info* info);

/* ---- full-mode overlap feedback (twolevel.py:186-239) as a dense global load: the
 *      capacity-difference, conductivity-gradient and source-scaling terms of the local
 *      field over the global quadrature points inside the local box.  src: the global
 *      Gaussian at t1 (or NULL / on = 0). */
int32_t tl_overlap_feedback_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                                 const double* local_new, const double* local_old, double dt,
                                 const tl_vc_material* mat_global, const tl_vc_material* mat_local,
                                 const tl_gaussian* src, double* load_out);

/* Same pass for the monolithic reference of a two-material setup (runner.py:141-151):
 * region = {lo[3], hi[3]}; tets whose centroid lies in the closed region use mat, the others
 * mat_outside (PiecewiseMaterial, materials.py:161-190; NULL: mat everywhere);
 * latent_inside_only != 0 restricts the latent term to the region (latent_reference local). */
int32_t tl_vc_step_region_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                               const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                               const double* T_lag, const double* extra_load, const tl_gaussian* src,
                               const tl_robin* robin, const uint8_t* dirichlet_mask, const double* g, double rtol,
                               int32_t maxiter, double* x_out, tl_solve_info* info);

/* The whole Picard loop of a nonlinear step on the device (fem.py:307-355): passes of
 * tl_vc_step_region_host starting from T_lag = T_old, the relative increment
 * ||x - T_lag|| / ||x|| reduced on the device, lag damping theta halved (>= 0.25) when the
 * increment stalls (>= 0.9 of the previous).  Stops when linear != 0 (one pass), when the
 * increment drops below picard_tol, after picard_max passes, or at the first pass whose CG
 * fails (info->status != TL_SOLVE_OK).  passes / pass_iters[picard_max] / pass_ms[picard_max]
 * report the passes, their CG iterations and PCG launch times; inc_out the last increment
 * (the caller raises NonConvergence("Picard iteration", ...) when passes == picard_max and
 * inc_out >= picard_tol). */
int32_t tl_vc_picard_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                          const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                          const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                          const uint8_t* dirichlet_mask, const double* g, double rtol, int32_t maxiter, int32_t linear,
                          double picard_tol, int32_t picard_max, double* x_out, int32_t* passes, int32_t* pass_iters,
                          float* pass_ms, double* inc_out, tl_solve_info* info);

/* tl_vc_picard_host with the Dirichlet data as a node list (fem.py:294-305 constrains the
 * listed nodes): dirichlet_nodes[n_dirichlet] (node ids) and dirichlet_values[n_dirichlet]
 * are scattered into the mask / value arrays on the device, so the call uploads
 * O(n_dirichlet) bytes of boundary data instead of 9 bytes per node. */
int32_t tl_vc_picard_nodes_host(const tl_grid_desc* grid, const tl_vc_material* mat, const tl_vc_material* mat_outside,
                                const double* region, int32_t latent_inside_only, double dt, const double* T_old,
                                const double* extra_load, const tl_gaussian* src, const tl_robin* robin,
                                const int32_t* dirichlet_nodes, int64_t n_dirichlet, const double* dirichlet_values,
                                double rtol, int32_t maxiter, int32_t linear, double picard_tol, int32_t picard_max,
                                double* x_out, int32_t* passes, int32_t* pass_iters, float* pass_ms, double* inc_out,
                                tl_solve_info* info);

/* ---- Fields kept on the device between step-level calls.
 * Every FIELD argument of the *_host entry points above and below (T_old, extra_load, g,
 * values, local_values, load_out, x_out, a, b, ...: the arrays with one entry per grid
 * node) may be a host pointer or a device pointer; unified virtual addressing tells them
 * apart.  A caller that holds the reference's FieldState values in device vectors
 * (tl_dev_alloc) therefore chains tl_vc_picard_nodes_host / tl_step_host /
 * tl_interpolate_nodes_host / tl_transmission_host / tl_overlap_feedback_host with no
 * per-node PCIe traffic.  tl_host_traffic reports the bytes that did cross (fields given as
 * host pointers, tl_dev_copy), optionally resetting the counters. */
int32_t tl_dev_alloc(int64_t bytes, void** out);
int32_t tl_dev_free(void* p);
int32_t tl_dev_copy(void* dst, const void* src, int64_t bytes);      /* any direction, complete on return */
int32_t tl_host_traffic(int64_t* h2d_bytes, int64_t* d2h_bytes, int32_t reset);
/* y = a x + y over n doubles (sums of interface loads, twolevel.py:254-262) */
int32_t tl_axpy_host(int64_t n, double a, const double* x, double* y);
/* Mesh.interpolate of the global field at listed nodes of the target lattice: the trace on
 * the interface nodes (twolevel.py:130-142); bitwise the values tl_interpolate_host writes
 * at those nodes. */
int32_t tl_interpolate_nodes_host(const tl_grid_desc* global_grid, const double* values, const tl_grid_desc* target,
                                  const int32_t* nodes, int64_t n, double* out);

/* Device time (CUDA events) of the last tl_vc_step_host's Jacobi-PCG launch (benchmark). */
int32_t tl_vc_last_cg_ms(float* ms);

/* ---- transmission_load (twolevel.py:159-183) for constant conductivities:
 *      load_out (dense, global nodes) = sum over the local grid's interface facets
 *      (LATERAL + BOTTOM, mesh.py:477-523) of jump * dT_local/dn * w_global at 3
 *      edge-midpoint quadrature points per facet; jump = kappa_global - kappa_local.
 *      Deterministic scatter (stable sort by node + ordered sums). */
int32_t tl_transmission_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                             const double* local_values, double jump, double* load_out);
/* Same with temperature-dependent conductivities: jump = kappa_g(T_qp) - kappa_l(T_qp),
 * T_qp the local P1 value at the quadrature point (twolevel.py:174-175). */
int32_t tl_transmission_tables_host(const tl_grid_desc* global_grid, const tl_grid_desc* local_grid,
                                    const double* local_values, const double* kg_T, const double* kg_v, int32_t nkg,
                                    const double* kl_T, const double* kl_v, int32_t nkl, double* load_out);

/* ---- discrete L2 norms with the P1 mass matrix (fem.mass_matrix / l2_norm,
 *      fem.py:434-446): out[0] = (a-b)^T M (a-b) (a^T M a when b == NULL),
 *      out[1] = b^T M b (0 when b == NULL). */
int32_t tl_mass_norms_host(const tl_grid_desc* grid, const double* a, const double* b, double* out);

/* ---- masked mass norms (twolevel.masked_mass, twolevel.py:361-373): out[0] = d^T M_in d,
 *      out[1] = d^T M_out d, d = a - b, M_in over the tets whose centroid lies in the closed
 *      box [box_lo, box_hi] (consistency_diagnostic, twolevel.py:376-400). */
int32_t tl_mass_norms_split_host(const tl_grid_desc* grid, const double* a, const double* b, const double* box_lo,
                                 const double* box_hi, double* out);

/* ---- error_metrics' per-record term (metrics.py:141-150): the reference field on
 *      ref_grid interpolated at grid's nodes (Mesh.interpolate), then
 *      out[0] = d^T M d with d = values - P1(ref), out[1] = P1(ref)^T M P1(ref). */
int32_t tl_error_l2_host(const tl_grid_desc* ref_grid, const double* ref_values, const tl_grid_desc* grid,
                         const double* values, double* out);

/* ---- deposit scatter: SweptTrackDeposit.load (sources.py:164-172), deterministic. */
int32_t tl_deposit_host(const tl_grid_desc* grid, const double* points, const double* power,
                        int32_t count, double* load_out);

/* ---- device-resident two-level run (run_spacetime / run_space hot loop). */
int32_t tl_run_create(const tl_run_desc* desc, tl_run** out);
int32_t tl_run_destroy(tl_run* run);
/* initial_state (twolevel.py:145-156): global = T0 everywhere, local = P1(global),
 * trace = P1(global) on gamma.  Resets the local box to the initial placement of the
 * run's descriptor, so a run can be reused for another schedule of the same problem. */
int32_t tl_run_initial(tl_run* run, double T0);
/* Upload a global field and re-derive local field + trace (initial_state with a
 * non-uniform T0). */
int32_t tl_run_set_global(tl_run* run, const double* Tg_host, int64_t n);
/* Run nsteps macro steps.  deposit arrays hold all samples referenced by the
 * plans (points xyz interleaved).  Solve outcomes are appended to the run's
 * info log (tl_run_take_info). */
int32_t tl_run_macro_steps(tl_run* run, const tl_macro_plan* plans, int32_t nsteps,
                           const tl_micro_plan* micro, int32_t nmicro,
                           const double* dep_points, const double* dep_power, int32_t ndep);
/* Batched runs (BASELINE config 5; runner.py:376-380 is the reference's concurrency point):
 * ONE macro step of `nruns` (<= 64) runs on one device whose local grids have one shape.
 * plans[r] is run r's macro plan (record must be 0), micro[r] / nmicro[r] its micro plans,
 * dep_*[r] / ndep[r] its deposit samples.  The global parts run per run; the i-th micro
 * solve (and the corrector) of all runs is one batched streaming solve, the systems
 * advancing in lockstep with their own scalars, stop tests and iteration counts.  Enqueued
 * on runs[0]'s stream; the other runs' streams are ordered around it.  Outcomes go to each
 * run's info log as usual. */
int32_t tl_runs_macro_step(tl_run** runs, int32_t nruns, const tl_macro_plan* plans,
                           const tl_micro_plan* const* micro, const int32_t* nmicro,
                           const double* const* dep_points, const double* const* dep_power,
                           const int32_t* ndep);
/* Snapshots kept by the last macro step with plan.record = 1:
 * which 0 = predicted global field, 1 = local field after micro step `index`
 * (index == n_micro: corrector result). */
int32_t tl_run_get_snapshot(tl_run* run, int32_t which, int32_t index, double* host, int64_t n);
/* Block until the run's stream is idle. */
int32_t tl_run_sync(tl_run* run);
/* which: 0 = global field, 1 = local field, 2 = trace (dense local array). */
int32_t tl_run_get_field(tl_run* run, int32_t which, double* host, int64_t n);
/* Selected entries of a field (which as above): host[e] = field[idx[e]], gathered on the device
 * so that only n values cross to the host (the interface trace of a run's final state,
 * InterfaceGamma.trace_nodes, mesh.py:507: ~2.6 % of the dense local array). */
int32_t tl_run_get_field_at(tl_run* run, int32_t which, const int32_t* idx, int64_t n, double* host);
/* Asynchronous read-back for pipelined callers (a recorder or a viewer consuming every
 * macro step while the next one computes).  Enqueues, in the run's stream order, a
 * device copy of the field into staging slot `slot` (0..3), then its transfer to `host`
 * on a separate copy stream, and returns at once; the run may go on with further macro
 * steps.  `host` should be pinned (page-locked) and must stay valid until
 * tl_run_field_wait(run, slot) returns. */
int32_t tl_run_field_async(tl_run* run, int32_t which, double* host, int64_t n, int32_t slot);
/* Block until the read-back enqueued on `slot` has landed in host memory. */
int32_t tl_run_field_wait(tl_run* run, int32_t slot);
/* Copy out (and clear) the per-solve info log; *count receives the number written. */
int32_t tl_run_take_info(tl_run* run, tl_solve_info* out, int32_t max, int32_t* count);
/* Melt-pool summary of both fields: max T and count of nodes with T > T_liquidus
 * (out: [gmax, lmax, gcount, lcount]).  Device reduction + 32-byte read. */
int32_t tl_run_melt_summary(tl_run* run, double T_liquidus, double* out4);
/* The run's CUDA stream (cudaStream_t) for event timing by the caller. */
int32_t tl_run_stream(tl_run* run, void** stream);
/* Number of kernels launched on the run's stream since creation. */
int64_t tl_run_launch_count(tl_run* run);
/* Per-launch CUDA-event timing of the solve kernel (k_pcg) on the run's stream.
 * When on, every solve launch is bracketed by an event pair; take_timing returns
 * (after a sync) the durations in ms and the level (0 global, 1 local) of the
 * launches since the last call, in launch order, with the number of solves each launch
 * ran (a persistent launch runs all micro solves of a macro step; the solve records of
 * tl_run_take_info are in the same order). */
int32_t tl_run_set_timing(tl_run* run, int32_t on);
int32_t tl_run_take_timing(tl_run* run, float* ms, int32_t* level, int32_t* nsolve, int32_t max,
                           int32_t* count);
/* Diagnostics: with TLGPU_PROF=1 in the environment the resident solve kernel records
 * %globaltimer stamps of CTA 0 at its phase boundaries (start, after the RHS, after
 * each of the two barriers of the first 64 iterations, end); this returns the stamps
 * of the most recent resident solve. */
int32_t tl_debug_profile(uint64_t* out, int32_t max, int32_t* count);
/* Write a scratch buffer larger than L2 on the run's stream (bench hygiene). */
int32_t tl_run_flush_l2(tl_run* run);
/* Multi-GPU local-only runs (tl_run_desc.external_planes > 0): tl_run_macro_steps skips
 * the deposit and the global solve and runs the local part of each macro step (trace,
 * micro solves, corrector, relocation; multirate.py:129-162) against the global planes
 * placed with tl_run_put_global_planes.  tl_run_reanchor moves the local box to `offset`
 * (Mesh._offset) and re-derives the whole local field and its trace by P1 interpolation
 * of the current global planes: relocate_local's field transfer (scanpath.py:243-248), or
 * initial_state (twolevel.py:145-156) at a later macro step. */
int32_t tl_run_reanchor(tl_run* run, const double* offset);
/* Copy device planes [k0, k1) of the global field (plane k0 first) into the run
 * (device-to-device on the run's stream; src must be ready when the call is made). */
int32_t tl_run_put_global_planes(tl_run* run, const double* src, int32_t k0, int32_t k1);

/* ---- multi-GPU: z-slab decomposition of the global solve ----------------
 * Replaces, per rank, the share of the global backward-Euler step
 * (twolevel.solve_global, lpbfsim/twolevel.py:242-271 -> fem.step_backward_euler,
 * fem.py:307-355 -> scipy cg, fem.py:271-298) that falls on the rank's node planes.
 * The reference has no decomposition.  The CG loop is DEVICE-RESIDENT: every scalar
 * (alpha, beta, the stop test) is computed by the kernels from the all-gathered partial
 * sums, so the host enqueues kernels and collectives without reading anything back:
 *   begin -> [all-gather sums] -> halo r -> loop { direction -> [all-gather] ->
 *   update(0) -> halo r (comm stream) || update(1) -> [all-gather] } -> halo x ->
 *   residual -> [all-gather] -> finish -> poll
 * The host enqueues a predicted number of iterations; iterations after the stop test
 * fired, and residual / finish before it fired, are no-ops; poll (the only host
 * synchronisation of a solve) reports whether finish has run.
 * Rank owns node planes [k0, k1) and stores planes [h0, h1) = [max(k0-1,0), min(k1+1,nz+1)):
 * x, b, r, p0, p1, load are device arrays of (h1-h0)*(nx+1)*(ny+1) doubles, plane h0
 * first, allocated so that the address of global node 0 (x - h0*(nx+1)*(ny+1)) is 16-byte
 * aligned and one element before / two after the stored range are readable (the bulk
 * copies round node ranges to 16 bytes).  sums: this rank's 8 partial sums (slot 0 r.r,
 * 1 r.z, 2 p.q, 3 ||Ax-b||^2, 4 non-finite count) — the all-gather's input; gath:
 * world x 8 doubles, every rank's sums in rank order — its output (NULL when world == 1).
 * work must hold tl_slab_work_len() doubles, zeroed once before first use.  Only
 * TL_DIRICHLET_BOTTOM is supported. */
typedef struct {
    tl_grid_desc grid;        /* the whole global grid                           */
    int32_t dirichlet_kind;   /* TL_DIRICHLET_BOTTOM                             */
    int32_t k0, k1;           /* owned node planes                               */
    double kappa, rho_c, dt;
    double g_const;           /* Dirichlet value (build-plate temperature)       */
    double* x;                /* T_old in (own planes), solution out, in place   */
    double *b, *r, *p0, *p1;  /* CG workspace                                    */
    const double* load;       /* deposit load or NULL                            */
    double* work;
    double* sums;             /* 8 doubles                                       */
    const double* gath;       /* world x 8 doubles (NULL: world == 1)            */
    int32_t world;
    int32_t maxiter;          /* scipy's maxiter (fem.py:285: 20 n)              */
    double rtol;              /* SolverSettings.linear_tol                       */
    void* stream;             /* cudaStream_t, NULL = legacy default stream      */
} tl_slab;

int64_t tl_slab_work_len(void);
/* Control-block reset + RHS (mass T_old + load [+ Gaussian] + Dirichlet lift), r = b,
 * x = 0 on own planes; sums[0] = b.b, sums[1] = r.z. */
int32_t tl_slab_begin(const tl_slab* s, const tl_gaussian* src);
/* scipy's stop test on the gathered sums; p = z (first) or beta p + z on stored planes;
 * sums[2] = p.Ap over own planes (bulk-copy z-march sweep). */
int32_t tl_slab_direction(const tl_slab* s);
/* x += alpha p, r -= alpha A p; part 0: the own planes a neighbour reads (their r is
 * what the halo exchange sends), part 1: the rest (sums[0] = r.r, sums[1] = r.z over all
 * own planes, iteration count + 1). */
int32_t tl_slab_update(const tl_slab* s, int32_t part);
/* After the stop test: ||A x - b||^2 and the non-finite count over own planes (x halo
 * must be current). */
int32_t tl_slab_residual(const tl_slab* s);
/* After the stop test: x_D = b_D (fem.py:289-290) and the true-residual check
 * (fem.py:286-288) on the gathered residual sums. */
int32_t tl_slab_finish(const tl_slab* s);
/* Synchronise the slab's stream and read the control block: *state 0 = iterating, 1 =
 * stopped (residual / finish pending), 2 = finished; info receives the outcome. */
int32_t tl_slab_poll(const tl_slab* s, int32_t* state, tl_solve_info* info);
/* Swept-track deposit (SweptTrackDeposit.load, sources.py:164-172) into s->load on the
 * rank's own nodes: the previous call's nodes are zeroed, the new samples scattered with
 * Kuhn-P1 weights and merged in np.add.at order.  points (3 count) and power (count)
 * are DEVICE arrays; count <= 512. */
int32_t tl_slab_deposit(const tl_slab* s, const double* points, const double* power, int32_t count);

#ifdef __cplusplus
}
#endif
#endif /* TLGPU_H */
