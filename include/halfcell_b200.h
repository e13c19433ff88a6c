/*
 * halfcell_b200 — C ABI of the B200-native full-order implicit step of the
 * microstructure-resolved half-cell model (arXiv 1704.04139).
 *
 * Every entry point replaces one Python entry point of the reference package
 * `halfcell` (reference tree `pkg/src/halfcell/...`, cited as file:line).  The
 * ABI uses plain pointers and sizes only; device pointers are CUDA global
 * memory (e.g. `torch.Tensor.data_ptr()`), `stream` is a `cudaStream_t`
 * (NULL = legacy default stream).  All functions return HC_OK or an error code;
 * `hc_last_error()` returns the message of the last failure on the calling
 * thread.  Errors map 1:1 onto the reference exception classes
 * (`src/halfcell/errors.py:1-37`).
 *
 * Packed state layout follows the reference exactly (`fvm/operator.py:3-7`,
 * `fvm/dofmap.py:1-7`): x = [c-block (graphite + electrolyte voxels in flat
 * order), phi-block (all non-grounded voxels in flat order)], fp64.
 */
#ifndef HALFCELL_B200_H
#define HALFCELL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (reference errors.py) ---- */
#define HC_OK 0
#define HC_ERR_CUDA 1          /* CUDA runtime failure / no device            */
#define HC_ERR_MODEL 2         /* ModelError                                   */
#define HC_ERR_NUMERICS 3      /* NumericsError (non-finite operator value)    */
#define HC_ERR_NONCONVERGENCE 4/* NonConvergence (Newton / Krylov budget)      */
#define HC_ERR_ARGUMENT 5      /* ValueError / ConfigError                     */
#define HC_ERR_SIMULATION 6    /* SimulationError (time step underflow)        */
#define HC_ERR_REDUCTION 7     /* ReductionError (POD)                         */

#define HC_MAX_OCP 32
#define HC_ROM_MAX_K 160       /* reduced dimension limit (dense LU in shared memory) */

/* MaterialParams (echem/params.py:50-113) + PhysConstants (params.py:26-29). */
typedef struct hc_params {
  double temperature, d_gr, sigma_gr, sigma_li, sigma_cc, sigma_pl, d_el, kappa_el,
         t_plus, dlnf_dlnc, i00_grel, i00_ceel, i00_plel, c_gr_max,
         n_const_thickness, c_li_metal, faraday, gas_constant;
  int32_t n_ocp, pad_;
  double ocp_soc[HC_MAX_OCP];
  double ocp_v[HC_MAX_OCP];
} hc_params;

/* Sizes of an operator: Dofmap counts (dofmap.py:20-36) and face-list lengths
 * of SystemOperator (operator.py:186-219). */
typedef struct hc_info {
  int64_t nx, ny, nz, n_vox;
  int64_t n_c, n_p, n_plated, n_dirichlet;
  int64_t n_bv, n_ce, n_strip, n_elel, n_drive_faces;
  double h, face_area, voxel_volume, n_const, scale;
} hc_info;

/* SolverConfig (fvm/newton.py:20-51). */
typedef struct hc_solver_config {
  double newton_rtol, newton_atol;
  int32_t newton_max_iter, krylov_max_iter;
  double linear_rtol;
  double dt_init, dt_min, dt_max, grow_factor, shrink_factor;
  int32_t easy_iter_threshold, implicit_plated;
  /* Krylov tolerance of Newton iteration k: max(linear_rtol, linear_safety * tol / |F_k|),
   * i.e. never solve beyond what the nonlinear tolerance can use (0 = always linear_rtol). */
  double linear_safety;
} hc_solver_config;

/* Result record of one Newton solve / accepted time step.  status: HC_OK, or the error
 * code of this cell in a batch (hc_step_batch). */
typedef struct hc_newton_stats {
  int32_t n_iter, krylov_iters, retries, status;
  double norm0, norm_final, tol, dt_used, dt_next, clamped_loss;
} hc_newton_stats;

typedef struct hc_operator hc_operator;

const char* hc_last_error(void);
int hc_device_count(int* out);

/* build_dofmap (fvm/dofmap.py:71-101) + SystemOperator.__init__/_build
 * (fvm/operator.py:109-242): uploads labels [z][y][x] (uint8, host), numbers
 * the DOFs, classifies and compacts every voxel face on the device.  Raises the
 * reference's ModelErrors (no graphite, no foil, no electrolyte path, no
 * counter collector to ground, forbidden adjacency, kinetics on a grounded face). */
int hc_operator_create(const uint8_t* labels_host, int32_t nx, int32_t ny, int32_t nz,
                       double voxel_size_um, const hc_params* params, hc_operator** out);
int hc_operator_destroy(hc_operator* op);
int hc_operator_info(const hc_operator* op, hc_info* out);
/* SystemOperator(dofmap, params) on a geometry that build_dofmap already classified
 * (fvm/operator.py:109-119: the reference also keeps the Dofmap and only reads the material
 * parameters in its constructor): replaces the operator's material parameters.  The geometry
 * (DOF numbering, face lists, slots) does not depend on them; every parameter-dependent
 * cache (multigrid values, captured solver graphs) is dropped. */
int hc_operator_set_params(hc_operator* op, const hc_params* params);

/* Export index arrays in the reference's layout into host int64 buffers.
 * what: 0 c_dof[n_vox], 1 p_dof[n_vox], 2 plated_voxels[n_plated], 3 dirichlet[n_dirichlet],
 *       4 bv (4 x n_bv: xc_gr, xc_el, xp_gr, xp_el), 5 ce (3 x n_ce: xp_fo, xc_el, xp_el),
 *       6 strip (4 x n_strip: xp_pl, xc_el, xp_el, slot), 7 elel (4 x n_elel: xc_i, xc_j, xp_i, xp_j)
 * (operator.py:188-219 attribute names). */
int hc_operator_export(const hc_operator* op, int32_t what, int64_t* host_out);

/* SystemOperator.apply and its parts (operator.py:331-389).  part:
 * 0 apply (full), 1 apply_bv, 2 apply_one_over_c, 3 apply_lin, 4 apply_const, 5 apply_bnd.
 * x, n_pl, out: device fp64, packed layout. */
int hc_apply(hc_operator* op, int32_t part, const double* x, const double* n_pl, double mu,
             double beta, double* out, void* stream);

/* Matrix-free Jacobian-vector product (jacobian(x) + diag(inv_dt on c rows)) @ v,
 * i.e. the matrix newton.py:126 factorizes, applied to v (operator.py:458-471). */
int hc_jvp(hc_operator* op, const double* x, const double* n_pl, double beta, double inv_dt,
           const double* v, double* out, void* stream);

/* Sparse Jacobian pattern (operator.py:458-471, CSR after duplicate summation)
 * for sparsity parity: fills *nnz when row_ptr == NULL, else row_ptr[n_total+1],
 * col_idx[nnz] (host int64) and optionally values (host fp64, at state x/n_pl/beta). */
int hc_jacobian_csr(hc_operator* op, const double* x, const double* n_pl, double beta,
                    int64_t* nnz, int64_t* row_ptr, int64_t* col_idx, double* values);

/* SystemOperator.A_lin (operator.py:221): the affine part's matrix in CSR, same calling
 * convention as hc_jacobian_csr (two calls: size, then fill). */
int hc_lin_csr(hc_operator* op, int64_t* nnz, int64_t* row_ptr, int64_t* col_idx, double* values);

/* SystemOperator.strip_face_currents (operator.py:391-399): the stripping current (A/m^2)
 * of every stripping face in the reference's face order, at packed state x (device) and
 * plated inventory n_pl, with the implicit-inventory coupling beta; out[n_strip] (device).
 * The matching plated slots are export selector 6, row 3. */
int hc_strip_face_currents(hc_operator* op, const double* x, const double* n_pl, double beta,
                           double* out, void* stream);

/* RestrictedSubOperator.apply / .jacobian (operator.py:541-646): selected output rows of
 * a nonlinear sub-operator evaluated from its stencil values only.  The face table is the
 * one the reduced model's online kernel reads (hc_rom): n_f faces with f_kind (0 BV,
 * 1 counter exchange, 2 stripping, 3 electrolyte-electrolyte), f_dof[n_f][4] stencil
 * positions, f_slot plated slots; rows as CSR row_ptr[n_rows+1] -> (row_face, row_coef).
 * x_st[n_s], n_pl (device); out[n_rows] (device) and, if jac != NULL, the dense local
 * Jacobian jac[n_rows][n_s] (device, row-major). */
int hc_restricted_eval(hc_operator* op, int32_t n_rows, int32_t n_f, int32_t n_s, const int32_t* f_kind,
                       const int32_t* f_dof, const int32_t* f_slot, const int32_t* row_ptr,
                       const int32_t* row_face, const double* row_coef, const double* x_st,
                       const double* n_pl, double beta, double* out, double* jac, void* stream);

/* newton_solve (fvm/newton.py:86-168): solves m (x - x_prev)/dt + A(x; mu) = 0
 * from x_guess; x_out receives the converged packed state (device). */
int hc_newton_solve(hc_operator* op, const double* x_guess, double dt, const double* x_prev,
                    const double* n_pl, double mu, const hc_solver_config* cfg, double* x_out,
                    hc_newton_stats* stats, void* stream);

/* newton_solve with its full signature and result (fvm/newton.py:86-168): `source`
 * (packed, device, may be NULL) is added to every residual (newton.py:107-108);
 * iterates[max_iterates][n_total] (device, may be NULL) receives every accepted Newton
 * iterate (NewtonResult.iterates) and norms[max_norms] (host, may be NULL) the residual
 * norm of the guess and of every iterate (NewtonResult.residual_norms); stats->n_iter
 * is the number of iterates. */
int hc_newton_solve_ex(hc_operator* op, const double* x_guess, double dt, const double* x_prev,
                       const double* n_pl, double mu, const hc_solver_config* cfg, const double* source,
                       double* iterates, int32_t max_iterates, double* norms, int32_t max_norms,
                       double* x_out, hc_newton_stats* stats, void* stream);

/* solve_initial_potential (fvm/newton.py:171-206): phi block at frozen c. */
int hc_solve_initial_potential(hc_operator* op, const double* x0, const double* n_pl, double mu,
                               const hc_solver_config* cfg, double* x_out, hc_newton_stats* stats,
                               void* stream);

/* step (fvm/timestepping.py:64-106): one accepted implicit-Euler step with
 * retry-on-failure, explicit plated-inventory update.  x and n_pl are updated
 * in place (device); stats carries dt_used / dt_next / retries / clamped loss. */
int hc_step(hc_operator* op, double* x, double* n_pl, double t, double dt_suggest, double mu,
            const hc_solver_config* cfg, hc_newton_stats* stats, void* stream);

/* hc_step that also returns the Newton iterates of the accepted solve (what step()
 * hands to observers' on_iterates, timestepping.py:98-101): iterates[max_iterates][n_total]
 * (device); stats->n_iter of them are written. */
int hc_step_ex(hc_operator* op, double* x, double* n_pl, double t, double dt_suggest, double mu,
               const hc_solver_config* cfg, double* iterates, int32_t max_iterates,
               hc_newton_stats* stats, void* stream);

/* Rebuild the multigrid preconditioner's Galerkin values at the next Newton iteration
 * (they are otherwise refreshed once every 32 Newton solves and on every dt change; the
 * Krylov method always applies the exact current Jacobian). */
int hc_precond_refresh(hc_operator* op);

/* Same step with HOST state buffers: copies in, steps on the device, copies out
 * (the reference-facing end-to-end call used by bench.py's e2e leg). */
int hc_step_host(hc_operator* op, double* x_host, double* n_pl_host, double t, double dt_suggest,
                 double mu, const hc_solver_config* cfg, hc_newton_stats* stats);

/* Batched parameter study (BASELINE config 3): one accepted step for each of n
 * independent cells (own operator, state, dt, applied current) on the device;
 * cells run concurrently on their operators' private streams, driven by
 * n_threads host threads.  x[i], n_pl[i] are device pointers updated in place. */
int hc_step_batch(hc_operator* const* ops, int32_t n, double* const* x, double* const* n_pl,
                  const double* dt_suggest, const double* mu, const hc_solver_config* cfg,
                  hc_newton_stats* stats, int32_t n_threads);

/* POD snapshot Gram G = S^T diag(w) S for S (n_dof x n_snap, column-major,
 * device fp64) — the method-of-snapshots correlation matrix (SPEC mor.pod);
 * G is n_snap x n_snap column-major on the device.  w may be NULL (identity). */
int hc_pod_gram(const double* S, const double* w, int64_t n_dof, int64_t n_snap, double* G,
                void* stream);

/* The same Gram for S stored row-major (n_dof x n_snap, the snapshots of one DOF
 * contiguous — the layout a snapshot matrix filled column by column in a row-major
 * tensor has); no transpose copy. */
int hc_pod_gram_rows(const double* S, const double* w, int64_t n_dof, int64_t n_snap, double* G,
                     void* stream);

/* The dense contractions of the reduced-basis stage on the FP64 tensor cores (DMMA):
 * C[i][j] = sum_k w[k] A(k, i) B(k, j), i < M, j < N, k < K, with strided operands
 * A(k, i) = A[k sa_k + i sa_i], B(k, j) = B[k sb_k + j sb_j] (device fp64) and optional
 * weights w[K] (NULL = 1); C row-major with leading dimension ldc (device).  Covers the
 * POD projection S (U / sigma), the CholeskyQR solve V R^-1, the EI block update and
 * B^T W (SPEC mor.pod / build_rom; no counterpart in the reference tree). */
int hc_dgemm(const double* A, int64_t sa_k, int64_t sa_i, const double* B, int64_t sb_k, int64_t sb_j,
             const double* w, int64_t K, int32_t M, int32_t N, double* C, int64_t ldc, void* stream);

/* Measured FP64 tensor-core (DMMA) throughput of the device in TFLOP/s (register-only
 * probe kernel, CUDA events): the roofline denominator of the reduced-basis contractions. */
int hc_dmma_peak(double* tflops, void* stream);

/* Reduced-order model for the online stage (SPEC mor.build_rom / solve_rom; no
 * counterpart in the reference tree, whose mor package is not shipped).  All arrays are
 * device memory.  x = B x~ with B = blockdiag(V_c, V_phi); the first k_c reduced
 * coordinates belong to V_c.  Dense matrices are row-major. */
typedef struct hc_rom {
  int32_t k, k_c;     /* reduced dimension, c-block part                              */
  int32_t m;          /* empirical-interpolation rows (Eq. 16 points)                 */
  int32_t n_s;        /* stencil DOFs (full-order DOFs the EI rows and strip faces read) */
  int32_t n_f;        /* active faces                                                 */
  int32_t n_pl;       /* plated-lithium slots (inventory carried exactly)             */
  const double* A;    /* [k][k]  B^T A_lin B                                          */
  const double* Mr;   /* [k][k]  B^T diag(c rows) B (implicit-Euler mass)            */
  const double* bnd;  /* [k]     B^T b_bnd (per unit applied current)                 */
  const double* E;    /* [k][m]  B^T W (W_pi)^-1                                      */
  const double* BS;   /* [n_s][k] rows of B at the stencil DOFs                       */
  const int32_t* f_kind;  /* [n_f] 0 BV, 1 counter exchange, 2 stripping, 3 electrolyte-electrolyte */
  const int32_t* f_dof;   /* [n_f][4] stencil indices: BV (c_gr,c_el,phi_gr,phi_el), CE
                             (phi_fo,c_el,phi_el,-1), STRIP (phi_pl,c_el,phi_el,-1), ELEL
                             (c_i,c_j,phi_i,phi_j)                                   */
  const int32_t* f_slot;  /* [n_f] plated slot of a stripping face, else -1          */
  const int32_t* row_ptr; /* [m+1] CSR: EI row -> (face, coefficient)                  */
  const int32_t* row_face;
  const double* row_coef;
  const int32_t* pl_ptr;  /* [n_pl+1] CSR: plated slot -> its stripping faces         */
  const int32_t* pl_face;
  const double* q_v;      /* [k] B^T (cell-voltage functional)                        */
  const double* q_ac;     /* [k] B^T (mean solid concentration functional)            */
} hc_rom;

/* Reduced implicit-Euler trajectory (SPEC mor.solve_rom): n_steps fixed steps of size
 * dt at applied current mu from the reduced state xt[k] (updated in place) and the
 * plated inventory n_pl[n_pl] (updated in place), chord Newton with the reduced
 * Jacobian refreshed at the first iteration of every jac_steps-th step (and of a step
 * following one that needed more than `refresh` iterations) and every `refresh`
 * iterations inside a step, converged when each block's update is <= rtol relative.  qoi[2 n_steps] receives (cell voltage, mean
 * solid concentration) per step, iters[n_steps] the Newton iterations, xt_steps
 * [n_steps][k] (optional, may be NULL) the reduced state after every step (device).  One
 * kernel launch (one thread-block cluster) runs the whole loop.  HC_ERR_NONCONVERGENCE carries the failing step
 * in *failed_step. */
int hc_rom_run(hc_operator* op, const hc_rom* rom, double* xt, double* n_pl, double mu, double dt,
               int32_t n_steps, double rtol, int32_t max_iter, int32_t refresh, int32_t jac_steps,
               double* qoi, int32_t* iters, double* xt_steps, int32_t* failed_step, void* stream);

/* The same reduced trajectory for n_par parameter values at once (the MOR use case:
 * one thread-block cluster per value, all resident concurrently as far as the SMs
 * allow).  xt[n_par][k], n_pl[n_par][n_pl], mu[n_par] (device), qoi[n_par][2 n_steps],
 * iters[n_par][n_steps]; failed_step[n_par] (host) receives -1 or the failing step. */
int hc_rom_run_batch(hc_operator* op, const hc_rom* rom, int32_t n_par, double* xt, double* n_pl,
                     const double* mu, double dt, int32_t n_steps, double rtol, int32_t max_iter,
                     int32_t refresh, int32_t jac_steps, double* qoi, int32_t* iters, int32_t* failed_step,
                     void* stream);

/* Evict L2 by streaming a `bytes`-sized buffer through it (reads only, so no dirty
 * lines are left behind); used between timed iterations. */
int hc_flush_l2(int64_t bytes, void* stream);

/* Number of CUDA kernels this library has launched in the process (bench.py). */
int hc_launch_count(int64_t* out);

/* Average device time (ms, CUDA events on `stream`) of one launch of each
 * kernel of the residual and of J v at state x, with an L2 flush of
 * `flush_bytes` before every launch: ms_out[5] = {residual stencil, residual
 * interface faces, J v (fused stencil incl. interface faces), 0 (no separate
 * interface kernel), streaming copy of one double2 per voxel (calibration)}. */
int hc_time_kernels(hc_operator* op, const double* x, const double* n_pl, double beta,
                    double inv_dt, int32_t iters, int64_t flush_bytes, double* ms_out,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HALFCELL_B200_H */
