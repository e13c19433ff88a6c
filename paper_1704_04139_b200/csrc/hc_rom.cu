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
// the stencil, timestepping.py:260-267) and the two QoIs are recorded.  Nothing of
// full-order length is touched online; per-step cost depends on (k, M, |S|) only.
//
// One CTA of 1024 threads runs the loop (there is no grid-wide dependency to
// distribute at these sizes); every phase is separated by __syncthreads().
#include <cmath>

#include "hc_internal.cuh"

namespace hc {

enum : int32_t { RF_BV = 0, RF_CE = 1, RF_STRIP = 2, RF_ELEL = 3 };
constexpr int ROM_THREADS = 1024;

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

__global__ void __launch_bounds__(ROM_THREADS, 1)
k_rom_run(DevParams P, RomDev R, double* __restrict__ xt, double* __restrict__ npl, double mu, double dt,
          double face_area_over_F, int n_steps, double rtol, int max_iter, int refresh,
          double* __restrict__ xs, double* __restrict__ fq, double* __restrict__ fdq,
          double* __restrict__ G, double* __restrict__ qoi, int32_t* __restrict__ iters,
          int32_t* __restrict__ status) {
  extern __shared__ double sm[];
  const int k = R.k, m = R.m;
  double* J = sm;                 // [k][k] LU factors
  double* rr = J + k * k;         // [k] residual / Newton update
  double* xo = rr + k;            // [k] x~ at the start of the step
  double* nn = xo + k;            // [m] N at the EI rows
  double* red = nn + m;           // [64] reduction scratch
  int* piv = reinterpret_cast<int*>(red + 64);   // [k]
  const int tid = threadIdx.x, nt = blockDim.x;
  const double inv_dt = 1.0 / dt, beta = dt * face_area_over_F;

  auto eval_faces = [&](bool need_d) {
    for (int i = tid; i < R.n_s; i += nt) {   // x_S = B_S x~
      const double* b = R.BS + (long long)i * k;
      double s = 0.0;
      for (int j = 0; j < k; ++j) s = fma(b[j], xt[j], s);
      xs[i] = s;
    }
    __syncthreads();
    for (int f = tid; f < R.n_f; f += nt) {
      double q, d[4];
      const int sl = R.f_slot[f];
      rom_face(P, R.f_kind[f], xs, R.f_dof + 4 * f, sl >= 0 ? npl[sl] : 0.0, beta, &q, d);
      fq[f] = q;
      if (need_d)
        for (int c = 0; c < 4; ++c) fdq[4 * f + c] = d[c];
    }
    __syncthreads();
    for (int r = tid; r < m; r += nt) {
      double s = 0.0;
      for (int e = R.row_ptr[r]; e < R.row_ptr[r + 1]; ++e) s = fma(R.row_coef[e], fq[R.row_face[e]], s);
      nn[r] = s;
    }
    __syncthreads();
  };

  for (int step = 0; step < n_steps; ++step) {
    for (int j = tid; j < k; j += nt) xo[j] = xt[j];
    __syncthreads();
    bool conv = false;
    int it = 0;
    for (; it < max_iter && !conv; ++it) {
      const bool fresh = it == 0 || (refresh > 0 && it % refresh == 0);
      eval_faces(fresh);
      // r~ = M~ (x~ - x~_old)/dt + A~ x~ + mu b~ + E N
      for (int i = tid; i < k; i += nt) {
        const double* a = R.A + (long long)i * k;
        const double* mr = R.Mr + (long long)i * k;
        double s = mu * R.bnd[i];
        for (int j = 0; j < k; ++j) s = fma(a[j], xt[j], fma(mr[j] * inv_dt, xt[j] - xo[j], s));
        const double* e = R.E + (long long)i * m;
        for (int r = 0; r < m; ++r) s = fma(e[r], nn[r], s);
        rr[i] = s;
      }
      if (fresh) {
        // G = (dN/dx_S) B_S  (m x k), then J~ = M~/dt + A~ + E G, LU in shared memory
        for (int idx = tid; idx < m * k; idx += nt) {
          const int r = idx / k, j = idx - r * k;
          double s = 0.0;
          for (int e = R.row_ptr[r]; e < R.row_ptr[r + 1]; ++e) {
            const int f = R.row_face[e];
            double t = 0.0;
            for (int c = 0; c < 4; ++c) {
              const int d = R.f_dof[4 * f + c];
              if (d >= 0) t = fma(fdq[4 * f + c], R.BS[(long long)d * k + j], t);
            }
            s = fma(R.row_coef[e], t, s);
          }
          G[idx] = s;
        }
        __syncthreads();
        for (int idx = tid; idx < k * k; idx += nt) {
          const int i = idx / k, j = idx - i * k;
          double s = R.A[idx] + R.Mr[idx] * inv_dt;
          const double* e = R.E + (long long)i * m;
          for (int r = 0; r < m; ++r) s = fma(e[r], G[(long long)r * k + j], s);
          J[idx] = s;
        }
        __syncthreads();
        for (int c = 0; c < k; ++c) {   // LU with partial pivoting (column c)
          if (tid < 32) {
            double best = -1.0;
            int bi = c;
            for (int i = c + tid; i < k; i += 32) {
              const double v = fabs(J[i * k + c]);
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
              const double t = J[c * k + j];
              J[c * k + j] = J[p * k + j];
              J[p * k + j] = t;
            }
          __syncthreads();
          const double d = J[c * k + c];
          for (int idx = tid; idx < (k - c - 1) * (k - c); idx += nt) {
            const int i = c + 1 + idx / (k - c), j = c + idx % (k - c);
            const double l = J[i * k + c] / d;
            if (j == c) continue;
            J[i * k + j] = fma(-l, J[c * k + j], J[i * k + j]);
          }
          __syncthreads();
          for (int i = c + 1 + tid; i < k; i += nt) J[i * k + c] /= d;
          __syncthreads();
        }
      }
      __syncthreads();
      // solve J delta = r (pivots, forward, backward) on one warp, then x~ -= delta
      if (tid < 32) {
        for (int c = 0; c < k; ++c) {
          const int p = piv[c];
          if (p != c && tid == 0) {
            const double t = rr[c];
            rr[c] = rr[p];
            rr[p] = t;
          }
        }
        __syncwarp();
        for (int c = 0; c < k; ++c) {
          const double v = rr[c];
          for (int i = c + 1 + tid; i < k; i += 32) rr[i] = fma(-J[i * k + c], v, rr[i]);
          __syncwarp();
        }
        for (int c = k - 1; c >= 0; --c) {
          if (tid == 0) rr[c] /= J[c * k + c];
          __syncwarp();
          const double v = rr[c];
          for (int i = tid; i < c; i += 32) rr[i] = fma(-J[i * k + c], v, rr[i]);
          __syncwarp();
        }
      }
      __syncthreads();
      // convergence per block: |delta_c| <= rtol |x~_c| and |delta_p| <= rtol (|x~_p| + 1)
      if (tid < 32) {
        double dc = 0.0, xc = 0.0, dp = 0.0, xp = 0.0;
        for (int j = tid; j < k; j += 32) {
          const double d = rr[j], x = xt[j] - d;
          if (j < R.k_c) { dc += d * d; xc += x * x; } else { dp += d * d; xp += x * x; }
        }
        for (int o = 16; o; o >>= 1) {
          dc += __shfl_down_sync(0xffffffffu, dc, o);
          xc += __shfl_down_sync(0xffffffffu, xc, o);
          dp += __shfl_down_sync(0xffffffffu, dp, o);
          xp += __shfl_down_sync(0xffffffffu, xp, o);
        }
        if (tid == 0) {
          const bool ok = sqrt(dc) <= rtol * sqrt(xc) && sqrt(dp) <= rtol * (sqrt(xp) + 1.0);
          red[0] = ok ? 1.0 : 0.0;
          red[1] = (dc == dc && dp == dp) ? 1.0 : 0.0;
        }
      }
      __syncthreads();
      for (int j = tid; j < k; j += nt) xt[j] -= rr[j];
      conv = red[0] != 0.0;
      const bool finite = red[1] != 0.0;
      __syncthreads();
      if (!finite) {
        if (tid == 0) { status[0] = 2; status[1] = step; }
        return;
      }
    }
    if (!conv) {
      if (tid == 0) { status[0] = 1; status[1] = step; }
      return;
    }
    // exact plated-inventory update at the converged state (n_pl is not reduced)
    eval_faces(false);
    for (int s = tid; s < R.n_pl; s += nt) {
      double flux = 0.0;
      for (int e = R.pl_ptr[s]; e < R.pl_ptr[s + 1]; ++e) flux += fq[R.pl_face[e]] / P.sc * face_area_over_F;
      npl[s] = fmax(npl[s] - dt * flux, 0.0);
    }
    if (tid < 32) {   // QoIs are linear functionals of x~
      double v = 0.0, c = 0.0;
      for (int j = tid; j < k; j += 32) {
        v = fma(R.q_v[j], xt[j], v);
        c = fma(R.q_ac[j], xt[j], c);
      }
      for (int o = 16; o; o >>= 1) {
        v += __shfl_down_sync(0xffffffffu, v, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
      }
      if (tid == 0) {
        qoi[2 * step] = v;
        qoi[2 * step + 1] = c;
        iters[step] = it;
      }
    }
    __syncthreads();
  }
  if (tid == 0) { status[0] = 0; status[1] = n_steps; }
}

void rom_run(const Operator& op, const hc_rom* rom, double* xt, double* npl, double mu, double dt,
             int32_t n_steps, double rtol, int32_t max_iter, int32_t refresh, double* qoi,
             int32_t* iters, int32_t* status_host, cudaStream_t s) {
  RomDev R{rom->k, rom->k_c, rom->m, rom->n_s, rom->n_f, rom->n_pl, rom->A, rom->Mr, rom->bnd,
           rom->E, rom->BS, rom->row_coef, rom->q_v, rom->q_ac, rom->f_kind, rom->f_dof, rom->f_slot,
           rom->row_ptr, rom->row_face, rom->pl_ptr, rom->pl_face};
  if (R.k < 1 || R.k > HC_ROM_MAX_K || R.m < 0 || R.n_s < 0 || R.n_f < 0 || R.k_c < 0 || R.k_c > R.k)
    throw Error(HC_ERR_ARGUMENT, "reduced model dimensions out of range");
  DBuf<double> xs(std::max(R.n_s, 1)), fq(std::max(R.n_f, 1)), fdq(4LL * std::max(R.n_f, 1)),
      G((long long)std::max(R.m, 1) * R.k);
  DBuf<int32_t> st(2);
  const size_t smem = ((size_t)R.k * R.k + 2 * R.k + R.m + 64) * sizeof(double) + R.k * sizeof(int);
  HC_CUDA(cudaFuncSetAttribute(k_rom_run, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double fa_F = op.info.face_area / op.host_params.faraday;
  k_rom_run<<<1, ROM_THREADS, smem, s>>>(op.P, R, xt, npl, mu, dt, fa_F, n_steps, rtol, max_iter, refresh,
                                         xs.p, fq.p, fdq.p, G.p, qoi, iters, st.p);
  HC_COUNT();
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaMemcpyAsync(status_host, st.p, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hc
