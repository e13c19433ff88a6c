// Aggregation multigrid data structures (see hc_amg.cu).
#pragma once

#include "hc_internal.cuh"

#define HC_COARSE_MAX 160    /* largest coarsest level inverted in shared memory (one CTA) */
#define HC_COARSE_CAP 4096   /* largest dense coarsest level at all (blocked Gauss-Jordan in global memory) */

namespace hc {

// element type of the coarse-level cycle vectors (levels >= 1: iterates, right-hand
// sides, residuals, D^-1); sums are accumulated in fp64, the vectors stored in fp32 (the
// preconditioner needs no more; the Krylov method works in fp64)
using CV = double;

struct Csr {
  int n = 0;
  long long nnz = 0;
  DBuf<int32_t> rp, ci;
  DBuf<double> v;
  DBuf<float> vf;    // fp32 copy used by the cycle's sweeps (the preconditioner needs no fp64)
  // sliced-ELL copy for the sweeps (rows in slices of 32 = one warp, each slice padded to
  // its longest row and stored column-major): the k-th entries of 32 consecutive rows are
  // read by one coalesced load, and their columns are mostly consecutive, so the x gathers
  // touch few sectors.  Padding entries hold column = row and value 0.
  int sl_n = 0;                    // rows (0: no sliced copy)
  int sl_t = 1;                    // lanes per row
  DBuf<int32_t> sl_ptr, sl_col;    // slice offsets [n / 32 + 1], columns
  DBuf<int32_t> sl_map;            // CSR position of every sliced entry, -1 for padding
  DBuf<float> sl_vf;               // values, gathered from vf after every numeric setup
  long long sl_nnz = 0;
  // packed copy for the sweeps (levels >= 1): one 32-bit word per entry = bf16 value << 16 |
  // 16-bit column offset from the row's (CSR) or slice's (sliced ELL) smallest column; the
  // diagonal entry holds value 0 and the diagonal is kept per row in fp32, with the rounding
  // errors of the row's off-diagonal entries added to it, so every row sum is preserved
  // (half the bytes per entry; Krylov counts unchanged, profiles/r02_amg_packed_ab.txt)
  bool pk_ok = false;                  // every row / slice spans fewer than 65536 columns
  DBuf<int32_t> pk_base, sl_base;      // smallest column per row / per slice
  DBuf<uint16_t> pk_off, sl_off;       // static column offsets per entry (pattern only)
  DBuf<uint32_t> pk, sl_pk;            // packed entries (values refreshed with the hierarchy)
  DBuf<float> pk_diag;                 // compensated diagonal per row
};

struct AmgLevel {
  int n = 0;                             // rows (level 0: one per voxel, empty outside the field)
  Csr A;                                 // level operator (level 0 only feeds the Galerkin product)
  DBuf<double> dinv;
  DBuf<int32_t> parent;                  // tentative aggregate of each row, -1 if empty
  bool smoothed = false;                 // P is a smoothed (not tentative) prolongator
  bool filtered = false;                 // ... smoothed with the filtered (strong-graph) operator
  Csr P;                                 // prolongator to the next level (smoothed aggregation)
  Csr AP;                                // A P (Galerkin intermediate)
  Csr R;                                 // P^T A for a tentative P (levels >= 1): the member-row
                                         // sums, so b_next = P^T b - R x is one pass (no residual vector)
  DBuf<int32_t> pt_ptr, pt_row, pt_idx;  // P^T: for each coarse unknown, (row, value index) pairs
  DBuf<double> ptv;                      // P^T values (gathered after every setup)
  DBuf<float> ptvf;                      // fp32 copy used by the cycle's restriction
  DBuf<CV> x, x2, b, res, acc;           // cycle vectors (levels >= 1)
  DBuf<CV> dinvc;                        // D^-1 for the cycle (levels >= 1)
  // sparsified sweep operator (levels >= 1 with long rows): the entries with |a_ij| >=
  // sparsify * |a_ii| at the first numeric setup keep their place, everything else is lumped
  // onto the diagonal at every setup (row sums preserved).  Only the sweeps read it (packed
  // copies only); the Galerkin products keep the full pattern.
  bool sp_ok = false;
  Csr As;                                // rp / ci of the kept pattern + packed copies
  DBuf<uint8_t> sp_keep;                 // per entry of A: kept (1) or lumped (0)
};

// device view of one CSR level for the cluster-fused coarse cycle (hc_amg.cu)
struct CoarseLev {
  int n;
  const int32_t *rp, *ci;
  const float* vf;              // fp32 values (or null: vd)
  const double* vd;
  const CV* dinv;
  CV *b, *x, *x2, *res;
  int tentative;                // prolongator is the tentative one (one entry of 1 per row)
  const int32_t* parent;
  const int32_t *prp, *pci;
  const double* pv;
  const int32_t *pt_ptr, *pt_row;
  const double* ptv;
};

struct AmgBlock {
  int nu = 1, nu_c = 2, pre_c = 2, post_c = 2;   // fine / CSR-level smoothing sweeps of this block (from Amg, HC_AMG_NU*_C0 override the c block)
  int field = 0;                  // 0: c block of T J, 1: phi block of J
  double alpha = 1.0;             // coarse-correction scaling
  std::vector<AmgLevel> levels;   // levels[0] is the fine grid
  bool sp_done = false;           // the sparsified sweep patterns were decided (first numeric setup)
  DBuf<double> dense, dense_inv;  // coarsest matrix and its inverse
  DBuf<double> gj_aug, gj_col, gj_row, gj_piv;   // blocked Gauss-Jordan work space (coarsest levels above HC_COARSE_MAX rows)
  int fuse_from = -1;             // levels >= fuse_from run as one cluster kernel (-1: none)
  DBuf<CoarseLev> clev;           // their device views
};

struct AmgGraph {
  const double2* r = nullptr;
  double2* z = nullptr;
  int mode = 0;
  bool presplit = false;
  double inv_dt = 0.0;
  cudaGraphExec_t exec = nullptr;
  unsigned long long n_kernels = 0;
};

struct Amg {
  ~Amg();
  bool use_graphs = true;
  std::vector<AmgGraph> graphs;
  AmgBlock blk[2];
  // coarsening stops at the first level with at most this many rows; that level is inverted densely
  // (<= HC_COARSE_MAX rows in shared memory, up to HC_COARSE_CAP by blocked Gauss-Jordan in global
  // memory) and every coarse solve is one dense mat-vec.  Measured against 128: the exact solve on a
  // few thousand rows replaces the 2-3 smallest levels' launch chains AND converges faster — tiny cell
  // 6.34 -> 3.3 ms per step (37.7 -> 15.6 BiCGStab iterations), medium 18.0 -> 13.7 (39.1 -> 32.5),
  // large 64.1 -> 59.8 (39.8 -> 36.9), batched 200 -> 269 cell-steps/s (48.5 -> 34.5)
  int coarse_max = 0;         // 0: by grid size, clamp(n_vox / 128, 1600, 4000) (HC_AMG_COARSE_MAX)
  int nu = 1;                // smoothing sweeps on the fine level (measured: 1 beats 2 on the medium cell)
  int nu_c = 2;              // smoothing sweeps on the CSR levels
  // smoothed transfers of the c block: -1 = by grid size, the first transfer on grids of at most 2 M
  // voxels (on top of the dense coarsest level: medium cell 13.6 -> 11.9 ms per step, 32.5 -> 27.1
  // iterations; tiny 2.90 -> 2.59 ms; batched 265 -> 315 cell-steps/s; the large cell's denser c level 1
  // costs more than its 36.4 -> 33.8 iterations save: 59.5 -> 62.5 ms, so plain aggregation there)
  int sa_levels_c = -1;
  double omega = 0.9;        // Jacobi smoothing weight
  // per-sweep weights (default omega): CSR-level zero-guess pre-sweep, first / second post-sweep;
  // fine-level pre (zero-guess) and post sweeps
  double w_pre = 0.9, w_post0 = 0.9, w_post1 = 0.9, wf_pre = 0.9, wf_post = 0.9, wf_post1 = 0.9;
  double omega_p = 2.0 / 3;  // prolongator smoothing weight
  int sa_levels = 2;         // smoothed prolongators on the first sa_levels transfers
  // transfers past the sa_levels smoothed ones are smoothed too when their fine level has
  // sa_rows_min..sa_rows rows (measured: medium cell, 10.6 k phi rows at level 2, 23.6 -> 15.6
  // BiCGStab iterations per step and 101 -> 118 steps/s; large cell, 13.5 k rows at level 3,
  // 36.3 -> 23.4 iterations and 13.4 -> 19.6 steps/s; its 83 k-row level 2 converges far worse
  // smoothed, and the batched cells' levels are below the window)
  int sa_rows_min = 8192, sa_rows = 32768;
  int sa_any = 1;            // 0: the size rule applies only to the transfer right after sa_levels
  double alpha = 1.0;
  int gamma = 1;             // cycles per coarse-level solve (2 = W-cycle)
  int wdepth = 3;
  int wmin = 1;
  int fuse_rows = 0;          // levels with at most this many rows ... (0: off, measured slower)
  long long fuse_nnz = 400000; // ... and nonzeros run as one cluster kernel (0 rows: off)
  bool fuse_restrict = true;  // residual + restriction as one pass on CSR levels (R = P^T A) ...
  bool fuse_restrict_sa = false;  // ... also where P is smoothed (HC_AMG_FUSE_RESTRICT_SA)
  int coarsen = 2;           // block growth factor of the transfers above level 1              // gamma cycles on CSR levels wmin..wdepth
  bool fp32_coarse = true;   // coarse-level sweeps read fp32 matrix values
  int sa_filter = 0;         // bit l: filtered smoothing of the phi transfer from level l
  double sparsify = 0.003;   // drop tolerance of the sparsified sweep operators (0: off; HC_AMG_SPARSIFY)
  int sparsify_min_rows = 1024;   // ... and at least this many rows (smaller levels are latency-bound)
  double sparsify_avg = 20;  // ... on levels with more nonzeros per row than this (HC_AMG_SPARSIFY_AVG)
  bool skip_planes = true;   // c-block fine sweeps only over the planes that hold c rows (HC_AMG_SKIP_PLANES)
  bool pack = true;          // packed (bf16 value | 16-bit column offset) level operators for the sweeps
  int sell_max_avg = 512;    // levels with at most this many nonzeros per row and at least
  int sell_min_rows = 131072; // sell_min_rows threads (rows x lanes per row) sweep through the
                              // sliced-ELL copy (0: off); measured at one lane per row: large cell
                              // 88.0 -> 83.7 ms per step, medium (70 k-row level) 20.2 -> 21.4 at 16 k;
                              // with 4 lanes per row on phi level 2 (183 nonzeros): 76.9 -> 75.7
  double sell_lane_nnz = 48;  // lanes per row: the smallest power of two with <= this many entries per lane
  int sell_force_t = 0;       // force the lanes per row (0: by the rule above)
  int refresh = 0;          // numeric setup every Newton iteration (1) or once per solve (0)
  int refresh_solves = 32;  // rebuild once every this many Newton solves (and when dt changes);
                            // 400-step medium / 200-step large runs: same Krylov totals as 8, 2-3 % faster
  long long solves = 0;
  double last_inv_dt = -1.0;
  bool force = false;        // rebuild at the next Newton iteration (after a stale-hierarchy Krylov failure)
  DBuf<double> rs[2], ea[2], eb[2], res, rc2;   // fine-level scalar vectors per block
  DBuf<double> res_c;                           // the c block's fine residual (block Jacobi)
  // block-Jacobi preconditioner (default): the two blocks' V-cycles are independent, so
  // the c-block cycle runs on a side stream (a parallel branch of the captured graph);
  // HC_AMG_BDIAG=0 restores block Gauss-Seidel (c right-hand side corrected by T J_cp e_phi)
  bool bdiag = true;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

Amg* build_amg(const Operator& op);
void amg_update(Operator& op, double inv_dt, int blocks, cudaStream_t s);  // blocks: 1 c, 2 phi
// presplit: the caller already wrote r's scalar right-hand sides (T r_c, r_phi) into
// rs[0], rs[1] (the Krylov vector kernels do, saving the split pass)
void amg_apply(Operator& op, const double2* r, double2* z, double inv_dt, int mode, cudaStream_t s,
               bool presplit = false);

}  // namespace hc
