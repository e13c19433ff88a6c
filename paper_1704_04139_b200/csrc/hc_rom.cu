// Reduced-order model, online stage (SPEC mor.solve_rom; arXiv 1704.04139 Eq. 20):
// implicit Euler + Newton in reduced coordinates, the whole time loop in ONE kernel.
//
// State x = B x~ with B = blockdiag(V_c, V_phi) (POD bases, orthonormal columns).
// Per Newton iteration:
//   x_S  = B_S x~                          (basis rows at the stencil DOFs only)
//   q_f, dq_f/dx for the active interface / electrolyte faces (BV, counter exchange,
//        stripping with the implicit plated inventory, chemical-potential faces)
//   N_pi = sum over each EI row's faces of coef * q_f          (Eq. 16 point values)
//   r~   = M~ (x~ - x~_old)/dt + A~ x~ + mu b~ + E N_pi         (E = B^T W (W_pi)^-1)
//   J~   = M~/dt + A~ + E (dN_pi/dx_S) B_S                      (chord: refreshed per step)
// then the dense k x k solve in shared memory (LU with partial pivoting).  After
// convergence the plated inventory is advanced exactly (all stripping faces are in
// the stencil, timestepping.py:50-57, 89-96) and the two QoIs are recorded.  Nothing of
// full-order length is touched online; per-step cost depends on (k, M, |S|) only.
//
// One thread-block cluster (16 CTAs of 1024 threads where the device schedules it,
// else 8) runs the loop: the stencil gathers, face kinetics, EI rows, the G and J~ rows
// are spread over the cluster's SMs, the dense LU / triangular solves run on CTA 0, and
// the phases are separated by cluster barriers (barrier.cluster, release/acquire).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "hc_internal.cuh"

namespace cg = cooperative_groups;

namespace hc {

enum : int32_t { RF_BV = 0, RF_CE = 1, RF_STRIP = 2, RF_ELEL = 3 };
constexpr int ROM_THREADS = 1024;
constexpr int TK = 16;    // E G panel depth
__host__ __device__ inline int rom_ld(int k) { return (k & 1) ? k : k + 1; }
constexpr int ROM_ACC = 4; // J~ entries per thread: k <= 160 rows over >= 8 CTAs

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct RomDev {
  int k, k_c, m, n_s, n_f, n_pl;
  const double *A, *Mr, *bnd, *E, *BS, *row_coef, *q_v, *q_ac;
  const int32_t *f_kind, *f_dof, *f_slot, *row_ptr, *row_face, *pl_ptr, *pl_face;
};

// face quantity q_f and its derivatives w.r.t. the face's (up to) four stencil DOFs;
// BV/CE/STRIP q = i / (F h) (operator.py:246-320), ELEL q = gX (log c_j - log c_i)
__device__ void rom_face(const DevParams& P, int kind, const double* xs, const int32_t* dof,
                         double npl, double beta, double* q, double* dq) {
  dq[0] = dq[1] = dq[2] = dq[3] = 0.0;
  if (kind == RF_BV) {   // (c_gr, c_el, phi_gr, phi_el)
    const double cg = xs[dof[0]], ce = xs[dof[1]], pg = xs[dof[2]], pe = xs[dof[3]];
    const double eta = pg - ocp_dev(cg, P) - pe;
    const double root = sqrt(cg * ce), sh = sinh(eta / P.vt), ch = cosh(eta / P.vt);
    *q = P.sc * 2.0 * P.i00_grel * root * sh;
    dq[0] = P.sc * 2.0 * P.i00_grel * (0.5 * sqrt(ce / cg) * sh - root * ch * ocp_slope_dev(cg, P) / P.vt);
    dq[1] = P.sc * P.i00_grel * sqrt(cg / ce) * sh;
    dq[2] = P.sc * 2.0 * P.i00_grel * root * ch / P.vt;
    dq[3] = -dq[2];
  } else if (kind == RF_CE) {   // (phi_foil, c_el, phi_el)
    const double pf = xs[dof[0]], pe = xs[dof[2]];
    *q = P.sc * 2.0 * P.i00_ceel * sinh((pf - pe) / P.vt);
    dq[0] = P.sc * 2.0 * P.i00_ceel * cosh((pf - pe) / P.vt) / P.vt;
    dq[2] = -dq[0];
  } else if (kind == RF_STRIP) {   // (phi_pl, c_el, phi_el)
    const double pp = xs[dof[0]], ce = xs[dof[1]], pe = xs[dof[2]];
    double dce = 0.0, dpp = 0.0;
    *q = P.sc * strip_current_dev(ce, pp, pe, npl, beta, P, &dce, &dpp);
    dq[0] = P.sc * dpp;
    dq[1] = P.sc * dce;
    dq[2] = -dq[0];
  } else {   // (c_i, c_j, phi_i, phi_j)
    const double ci = xs[dof[0]], cj = xs[dof[1]];
    *q = P.gX * (log(cj) - log(ci));
    dq[0] = -P.gX / ci;
    dq[1] = P.gX / cj;
  }
}

struct RomWork {
  double *x, *xs, *fq, *fdq, *nn, *rr, *G, *J, *npl, *qoi, *xt_steps;
  int32_t *iters, *status;
};

// acquire loads of values another CTA of the cluster wrote before the last cluster
// barrier (bypass the non-coherent L1)
__device__ __forceinline__ double ldc(const double* p) { return __ldcg(p); }

__global__ void __launch_bounds__(ROM_THREADS, 1)
k_rom_run(DevParams P, RomDev R, RomWork W, const double* __restrict__ mus, double dt, double face_area_over_F,
          int n_steps, double rtol, int max_iter, int refresh, int jac_steps) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), ncta = (int)cl.num_blocks();
  // one cluster per parameter value: shift every per-trajectory array to this one's slice
  const int par = (int)(blockIdx.x / ncta);
  const double mu = mus[par];
  {
    const long long k_ = R.k, m_ = max(R.m, 1);
    W.x += par * k_;
    W.xs += par * (long long)max(R.n_s, 1);
    W.fq += par * (long long)max(R.n_f, 1);
    W.fdq += par * 4LL * max(R.n_f, 1);
    W.nn += par * m_;
    W.rr += par * k_;
    W.G += par * m_ * k_;
    W.J += par * k_ * k_;
    W.npl += par * (long long)max(R.n_pl, 1);
    W.qoi += par * 2LL * max(n_steps, 1);
    W.iters += par * (long long)max(n_steps, 1);
    W.status += par * 4LL;
    if (W.xt_steps) W.xt_steps += par * (long long)max(n_steps, 1) * k_;
  }
  extern __shared__ double sm[];
  const int k = R.k, m = R.m;
  // [k][ld] LU factors (rank 0); odd row pitch so the column walks of the pivot search
  // and the triangular solves hit distinct shared-memory banks (a pitch of k doubles
  // put a warp's 32 rows on 2 banks: 16-way conflicts)
  const int ld = rom_ld(k);
  double* J = sm;
  double* rr = J + k * ld;        // [k] residual / Newton update (rank 0)
  double* xo = rr + k;            // [k] x~ at the start of the step
  double* red = xo + k;           // [64] reduction scratch
  double* sx = red + 64;          // [k] x~ (this CTA's copy)
  double* pg = sx + k;            // [TK][k] panel of G
  double* dgi = pg;               // [k] 1 / U_cc (rank 0; lives in the G panel, which is only
                                  // used before the factorization that rewrites it)
  int* piv = reinterpret_cast<int*>(pg + TK * k);   // [k]
  int* ctl = piv + k;             // [4] control broadcast inside the CTA
  int* perm = ctl + 4;            // [k] row permutation of the LU (all pivot swaps composed)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const int gtid = rank * nt + tid, gnt = ncta * nt;
  const int gw = rank * nwarp + warp, gnw = ncta * nwarp;
  const double inv_dt = 1.0 / dt, beta = dt * face_area_over_F;
  int* flag = W.status + 2;       // [2]: converged, finite (written by rank 0)

  auto load_x = [&]() {
    for (int j = tid; j < k; j += nt) sx[j] = ldc(W.x + j);
    __syncthreads();
  };
  // phases A-C: x_S = B_S x~, face quantities, N at the EI rows (and G when fresh)
  auto eval = [&](bool need_d, bool need_n) {
    for (int i = gw; i < R.n_s; i += gnw) {   // warp per row, coalesced
      const double* b = R.BS + (long long)i * k;
      double s = 0.0;
      for (int j = lane; j < k; j += 32) s = fma(b[j], sx[j], s);
      s = warp_sum(s);
      if (lane == 0) W.xs[i] = s;
    }
    cl.sync();
    for (int f = gtid; f < R.n_f; f += gnt) {
      const int* dof = R.f_dof + 4 * f;
      double xl[4];
      int dl[4] = {0, 1, 2, 3};
      for (int c = 0; c < 4; ++c) xl[c] = dof[c] >= 0 ? ldc(W.xs + dof[c]) : 1.0;
      double q, d[4];
      const int sl = R.f_slot[f];
      rom_face(P, R.f_kind[f], xl, dl, sl >= 0 ? ldc(W.npl + sl) : 0.0, beta, &q, d);
      W.fq[f] = q;
      if (need_d)
        for (int c = 0; c < 4; ++c) W.fdq[4 * f + c] = d[c];
    }
    cl.sync();
    if (!need_n) return;
    for (int r = gtid; r < m; r += gnt) {
      double s = 0.0;
      for (int e = R.row_ptr[r]; e < R.row_ptr[r + 1]; ++e) s = fma(R.row_coef[e], ldc(W.fq + R.row_face[e]), s);
      W.nn[r] = s;
    }
    if (need_d)   // G = (dN/dx_S) B_S  (m x k)
      for (int idx = gtid; idx < m * k; idx += gnt) {
        const int r = idx / k, j = idx - r * k;
        double s = 0.0;
        for (int e = R.row_ptr[r]; e < R.row_ptr[r + 1]; ++e) {
          const int f = R.row_face[e];
          double t = 0.0;
          for (int c = 0; c < 4; ++c) {
            const int d = R.f_dof[4 * f + c];
            if (d >= 0) t = fma(ldc(W.fdq + 4 * f + c), R.BS[(long long)d * k + j], t);
          }
          s = fma(R.row_coef[e], t, s);
        }
        W.G[idx] = s;
      }
    cl.sync();
  };

  load_x();
  int since = 0, prev_it = 0;
  for (int step = 0; step < n_steps; ++step) {
    for (int j = tid; j < k; j += nt) xo[j] = sx[j];
    __syncthreads();
    // chord Newton: the reduced Jacobian is refreshed at the first iteration of a step
    // every jac_steps steps (or after a slow step), and every `refresh` iterations
    bool step_fresh = step == 0 || since >= jac_steps || prev_it > refresh;
    bool conv = false;
    int it = 0;
    for (; it < max_iter && !conv; ++it) {
      const bool fresh = (it == 0 && step_fresh) || (refresh > 0 && it > 0 && it % refresh == 0);
      if (fresh) since = 0;
      eval(fresh, true);
      // phase D: r~ rows (warp per row) and, when fresh, J~ rows through G panels
      for (int i = gw; i < k; i += gnw) {
        const double* a = R.A + (long long)i * k;
        const double* mr = R.Mr + (long long)i * k;
        double s = 0.0;
        for (int j = lane; j < k; j += 32) s = fma(a[j], sx[j], fma(mr[j] * inv_dt, sx[j] - xo[j], s));
        const double* e = R.E + (long long)i * m;
        for (int r = lane; r < m; r += 32) s = fma(e[r], ldc(W.nn + r), s);
        s = warp_sum(s);
        if (lane == 0) W.rr[i] = s + mu * R.bnd[i];
      }
      if (fresh) {
        const int my_rows = (k - rank + ncta - 1) / ncta;   // rows i = rank + t ncta
        double acc[ROM_ACC] = {};
        for (int r0 = 0; r0 < m; r0 += TK) {
          const int tk = min(TK, m - r0);
          __syncthreads();
          for (int idx = tid; idx < TK * k; idx += nt) {
            const int r = idx / k;
            pg[idx] = r < tk ? ldc(W.G + (long long)(r0 + r) * k + (idx - r * k)) : 0.0;
          }
          __syncthreads();
#pragma unroll
          for (int h = 0; h < ROM_ACC; ++h) {
            const int idx = tid + h * nt;
            if (idx < my_rows * k) {
              const int i = rank + (idx / k) * ncta, j = idx % k;
              const double* e = R.E + (long long)i * m + r0;
              double a2 = 0.0;
              for (int r = 0; r < tk; ++r) a2 = fma(e[r], pg[r * k + j], a2);
              acc[h] += a2;
            }
          }
        }
#pragma unroll
        for (int h = 0; h < ROM_ACC; ++h) {
          const int idx = tid + h * nt;
          if (idx < my_rows * k) {
            const int i = rank + (idx / k) * ncta, j = idx % k;
            W.J[i * k + j] = R.A[i * k + j] + R.Mr[i * k + j] * inv_dt + acc[h];
          }
        }
      }
      cl.sync();
      // phase E (rank 0): LU when fresh, solve, update x~, convergence flags
      if (rank == 0) {
        if (fresh) {
          for (int idx = tid; idx < k * k; idx += nt) J[(idx / k) * ld + idx % k] = ldc(W.J + idx);
          __syncthreads();
          for (int c = 0; c < k; ++c) {   // LU with partial pivoting (column c)
            if (tid < 32) {
              double best = -1.0;
              int bi = c;
              for (int i = c + tid; i < k; i += 32) {
                const double v = fabs(J[i * ld + c]);
                if (v > best) { best = v; bi = i; }
              }
              for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_down_sync(0xffffffffu, best, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
              }
              if (tid == 0) piv[c] = bi;
            }
            __syncthreads();
            const int p = piv[c];
            if (p != c)
              for (int j = tid; j < k; j += nt) {
                const double t = J[c * ld + j];
                J[c * ld + j] = J[p * ld + j];
                J[p * ld + j] = t;
              }
            __syncthreads();
            const double d = J[c * ld + c];
            for (int idx = tid; idx < (k - c - 1) * (k - c); idx += nt) {
              const int i = c + 1 + idx / (k - c), j = c + idx % (k - c);
              if (j == c) continue;
              J[i * ld + j] = fma(-(J[i * ld + c] / d), J[c * ld + j], J[i * ld + j]);
            }
            __syncthreads();
            for (int i = c + 1 + tid; i < k; i += nt) J[i * ld + c] /= d;
            __syncthreads();
          }
          for (int c = tid; c < k; c += nt) dgi[c] = 1.0 / J[c * ld + c];   // U's reciprocal diagonal
          if (tid == 0) {   // the pivot swaps composed into one gather: rhs_perm[i] = rhs[perm[i]]
            for (int i = 0; i < k; ++i) perm[i] = i;
            for (int c = 0; c < k; ++c) {
              const int p = piv[c];
              if (p != c) { const int t = perm[c]; perm[c] = perm[p]; perm[p] = t; }
            }
          }
          __syncthreads();
        }
        if (tid < 32) {   // pivots, forward, backward on one warp
          // the pivot swaps were composed into one permutation at factorization time
          for (int j = tid; j < k; j += 32) rr[j] = ldc(W.rr + perm[j]);
          __syncwarp();
          // blocked by 32 columns: the sequential part of each diagonal block runs on
          // lane-resident values broadcast by shuffle, the rows outside it take the block's
          // 32 updates in one pass.  Every row receives its column updates in the same
          // (ascending / descending) column order as the plain column sweep.
          for (int b0 = 0; b0 < k; b0 += 32) {   // forward, unit lower L
            const int nbk = min(32, k - b0);
            double yb = tid < nbk ? rr[b0 + tid] : 0.0;
            for (int cc = 0; cc < nbk; ++cc) {
              const double l = (tid > cc && tid < nbk) ? J[(b0 + tid) * ld + b0 + cc] : 0.0;
              yb = fma(-l, __shfl_sync(0xffffffffu, yb, cc), yb);
            }
            if (tid < nbk) rr[b0 + tid] = yb;
            for (int i0 = b0 + nbk; i0 < k; i0 += 32) {
              const int i = i0 + tid;
              const bool ok = i < k;
              double acc = ok ? rr[i] : 0.0;
              for (int cc = 0; cc < nbk; ++cc) {
                const double l = ok ? J[i * ld + b0 + cc] : 0.0;
                acc = fma(-l, __shfl_sync(0xffffffffu, yb, cc), acc);
              }
              if (ok) rr[i] = acc;
            }
            __syncwarp();
          }
          for (int b0 = ((k - 1) / 32) * 32; b0 >= 0; b0 -= 32) {   // backward, U (1 / U_cc)
            const int nbk = min(32, k - b0);
            double yb = tid < nbk ? rr[b0 + tid] : 0.0;
            for (int cc = nbk - 1; cc >= 0; --cc) {
              if (tid == cc) yb *= dgi[b0 + cc];
              const double u = tid < cc ? J[(b0 + tid) * ld + b0 + cc] : 0.0;
              yb = fma(-u, __shfl_sync(0xffffffffu, yb, cc), yb);
            }
            if (tid < nbk) rr[b0 + tid] = yb;
            for (int i0 = 0; i0 < b0; i0 += 32) {
              const int i = i0 + tid;   // i < b0 always (b0 is a multiple of 32)
              double acc = rr[i];
              for (int cc = nbk - 1; cc >= 0; --cc)
                acc = fma(-J[i * ld + b0 + cc], __shfl_sync(0xffffffffu, yb, cc), acc);
              rr[i] = acc;
            }
            __syncwarp();
          }
          // convergence per block: |delta_c| <= rtol |x~_c|, |delta_p| <= rtol (|x~_p| + 1)
          double dc = 0.0, xc = 0.0, dp = 0.0, xp = 0.0;
          for (int j = tid; j < k; j += 32) {
            const double d = rr[j], x = sx[j] - d;
            if (j < R.k_c) { dc += d * d; xc += x * x; } else { dp += d * d; xp += x * x; }
          }
          dc = warp_sum(dc); xc = warp_sum(xc); dp = warp_sum(dp); xp = warp_sum(xp);
          for (int j = tid; j < k; j += 32) W.x[j] = sx[j] - rr[j];
          if (tid == 0) {
            flag[0] = sqrt(dc) <= rtol * sqrt(xc) && sqrt(dp) <= rtol * (sqrt(xp) + 1.0);
            flag[1] = dc == dc && dp == dp;
          }
        }
      }
      cl.sync();
      if (tid == 0) {
        ctl[0] = __ldcg(flag);
        ctl[1] = __ldcg(flag + 1);
      }
      load_x();   // (includes the CTA barrier that publishes ctl)
      conv = ctl[0] != 0;
      if (!ctl[1]) {
        if (rank == 0 && tid == 0) { W.status[0] = 2; W.status[1] = step; }
        return;
      }
    }
    if (!conv) {
      if (rank == 0 && tid == 0) { W.status[0] = 1; W.status[1] = step; }
      return;
    }
    ++since;
    prev_it = it;
    // exact plated-inventory update at the converged state (n_pl is not reduced)
    eval(false, false);
    for (int s = gtid; s < R.n_pl; s += gnt) {
      double flux = 0.0;
      for (int e = R.pl_ptr[s]; e < R.pl_ptr[s + 1]; ++e) flux += ldc(W.fq + R.pl_face[e]) / P.sc * face_area_over_F;
      W.npl[s] = fmax(ldc(W.npl + s) - dt * flux, 0.0);
    }
    if (rank == 0 && tid < 32) {   // QoIs are linear functionals of x~
      double v = 0.0, c = 0.0;
      for (int j = tid; j < k; j += 32) {
        v = fma(R.q_v[j], sx[j], v);
        c = fma(R.q_ac[j], sx[j], c);
      }
      v = warp_sum(v);
      c = warp_sum(c);
      if (tid == 0) {
        W.qoi[2 * step] = v;
        W.qoi[2 * step + 1] = c;
        W.iters[step] = it;
      }
      if (W.xt_steps)
        for (int j = tid; j < k; j += 32) W.xt_steps[(long long)step * k + j] = sx[j];
    }
    cl.sync();
  }
  if (rank == 0 && tid == 0) { W.status[0] = 0; W.status[1] = n_steps; }
}

void rom_run(const Operator& op, const hc_rom* rom, int n_par, double* xt, double* npl, const double* mus_dev,
             double dt, int32_t n_steps, double rtol, int32_t max_iter, int32_t refresh, int32_t jac_steps,
             double* qoi, int32_t* iters, double* xt_steps, int32_t* status_host, cudaStream_t s) {
  RomDev R{rom->k, rom->k_c, rom->m, rom->n_s, rom->n_f, rom->n_pl, rom->A, rom->Mr, rom->bnd,
           rom->E, rom->BS, rom->row_coef, rom->q_v, rom->q_ac, rom->f_kind, rom->f_dof, rom->f_slot,
           rom->row_ptr, rom->row_face, rom->pl_ptr, rom->pl_face};
  if (R.k < 1 || R.k > HC_ROM_MAX_K || R.m < 0 || R.n_s < 0 || R.n_f < 0 || R.k_c < 0 || R.k_c > R.k ||
      n_par < 1)
    throw Error(HC_ERR_ARGUMENT, "reduced model dimensions out of range");
  const long long np = n_par;
  DBuf<double> xs(np * std::max(R.n_s, 1)), fq(np * std::max(R.n_f, 1)), fdq(np * 4LL * std::max(R.n_f, 1)),
      nn(np * std::max(R.m, 1)), rr(np * R.k), G(np * std::max(R.m, 1) * R.k), J(np * R.k * R.k);
  DBuf<int32_t> st(np * 4);
  HC_CUDA(cudaMemsetAsync(st.p, 0, np * 4 * sizeof(int32_t), s));
  RomWork W{xt, xs.p, fq.p, fdq.p, nn.p, rr.p, G.p, J.p, npl, qoi, xt_steps, iters, st.p};
  const size_t smem = ((size_t)R.k * rom_ld(R.k) + 3 * R.k + 64 + (size_t)TK * R.k) * sizeof(double) +
                      (2 * R.k + 4) * sizeof(int);
  HC_CUDA(cudaFuncSetAttribute(k_rom_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  static int cluster = 0;   // largest cluster the device schedules (16 non-portable, else 8)
  if (!cluster) {
    cluster = 8;
    if (cudaFuncSetAttribute(k_rom_run, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(ROM_THREADS);
      q.dynamicSmemBytes = smem;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 16; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
      q.attrs = &at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_rom_run, &q) == cudaSuccess && n >= 1) cluster = 16;
    }
    cudaGetLastError();
    if (const char* e = getenv("HC_ROM_CLUSTER")) cluster = atoi(e) >= 16 ? 16 : 8;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cluster * n_par));
  cfg.blockDim = dim3(ROM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = cluster; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  const double fa_F = op.info.face_area / op.host_params.faraday;
  HC_CUDA(cudaLaunchKernelEx(&cfg, k_rom_run, op.P, R, W, mus_dev, dt, fa_F, (int)n_steps, rtol, (int)max_iter,
                             (int)refresh, (int)jac_steps));
  HC_COUNT();
  HC_CUDA(cudaMemcpyAsync(status_host, st.p, np * 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
}

// RestrictedSubOperator.apply / .jacobian (operator.py:598-646) from the same face
// table and face kinetics (rom_face) the online kernel evaluates its EI rows with:
// one thread per selected row, its faces in table order.
__global__ void k_restricted_eval(DevParams P, int n_rows, int n_s, const int32_t* __restrict__ f_kind,
                                  const int32_t* __restrict__ f_dof, const int32_t* __restrict__ f_slot,
                                  const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ row_face,
                                  const double* __restrict__ row_coef, const double* __restrict__ xs,
                                  const double* __restrict__ npl, double beta, double* __restrict__ out,
                                  double* __restrict__ jac) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  double acc = 0.0;
  for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
    const int f = row_face[e];
    const int32_t* dof = f_dof + 4 * f;
    const int sl = f_slot[f];
    double q, dq[4];
    rom_face(P, f_kind[f], xs, dof, sl >= 0 ? npl[sl] : 0.0, beta, &q, dq);
    const double c = row_coef[e];
    acc += c * q;
    if (jac)
      for (int j = 0; j < 4; ++j)
        if (dof[j] >= 0 && dq[j] != 0.0) jac[(long long)r * n_s + dof[j]] += c * dq[j];
  }
  out[r] = acc;
}

void restricted_eval(const Operator& op, int n_rows, int n_s, const int32_t* f_kind, const int32_t* f_dof,
                     const int32_t* f_slot, const int32_t* row_ptr, const int32_t* row_face,
                     const double* row_coef, const double* xs, const double* npl, double beta, double* out,
                     double* jac, cudaStream_t s) {
  if (n_rows <= 0) return;
  if (jac) HC_CUDA(cudaMemsetAsync(jac, 0, (size_t)n_rows * n_s * sizeof(double), s));
  k_restricted_eval<<<(n_rows + 127) / 128, 128, 0, s>>>(op.P, n_rows, n_s, f_kind, f_dof, f_slot, row_ptr,
                                                        row_face, row_coef, xs, npl, beta, out, jac);
  HC_COUNT();
  HC_CHECK_LAUNCH();
}

}  // namespace hc
