// Device-resident implicit step: preconditioned BiCGStab, damped Newton with
// positivity guard and line search, stationary potential solve, and the
// adaptive implicit-Euler step with the explicit plated-inventory update.
//
// Reference: fvm/newton.py:62-206, fvm/timestepping.py:50-106.
#include <chrono>
#include <cmath>
#include <algorithm>
#include <initializer_list>
#include <limits>

#include "hc_amg.cuh"
#include "hc_solver.cuh"

namespace hc {

namespace {
constexpr int TPB = 256;
inline int nblk(long long n, int tpb = TPB) { return (int)std::max<long long>(1, (n + tpb - 1) / tpb); }

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;
}

// partial dot products: out[blk] = <a,b>, out[nb + blk] = <c,d> (if c)
__global__ void k_dot2(long long n, const double2* __restrict__ a, const double2* __restrict__ b,
                       const double2* __restrict__ c, const double2* __restrict__ d,
                       double* __restrict__ part) {
  __shared__ double sh[32];
  double s1 = 0.0, s2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    s1 += x.x * y.x + x.y * y.y;
    if (c) {
      double2 u = c[i], w = d[i];
      s2 += u.x * w.x + u.y * w.y;
    }
  }
  s1 = block_sum(s1, sh);
  if (c) s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1;
    part[gridDim.x + blockIdx.x] = s2;
  }
}

// sums of squares of c and phi separately (NaN/Inf propagate)
__global__ void k_sumsq2(long long n, const double2* __restrict__ a, double* __restrict__ part) {
  __shared__ double sh[32];
  double s1 = 0.0, s2 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 x = a[i];
    s1 += x.x * x.x;
    s2 += x.y * x.y;
  }
  s1 = block_sum(s1, sh);
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s1;
    part[gridDim.x + blockIdx.x] = s2;
  }
}

__global__ void k_p_update(long long n, double beta, double omega, const double2* __restrict__ r,
                           const double2* __restrict__ v, double2* __restrict__ p) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 pi = p[i], ri = r[i], vi = v[i];
  p[i] = make_double2(ri.x + beta * (pi.x - omega * vi.x), ri.y + beta * (pi.y - omega * vi.y));
}

// y = a + alpha * b
__global__ void k_axpy(long long n, const double2* __restrict__ a, double alpha,
                       const double2* __restrict__ b, double2* __restrict__ y) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 u = a[i], w = b[i];
  y[i] = make_double2(u.x + alpha * w.x, u.y + alpha * w.y);
}

// x += alpha * p + omega * s
__global__ void k_x_update(long long n, double alpha, const double2* __restrict__ p, double omega,
                           const double2* __restrict__ s, double2* __restrict__ x) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 xi = x[i], pi = p[i], si = s[i];
  x[i] = make_double2(xi.x + alpha * pi.x + omega * si.x, xi.y + alpha * pi.y + omega * si.y);
}

__global__ void k_neg(long long n, const double2* __restrict__ a, double2* __restrict__ y) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 u = a[i];
  y[i] = make_double2(-u.x, -u.y);
}

__global__ void k_zero_c(long long n, double2* __restrict__ y) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) y[i].x = 0.0;
}

__global__ void k_extract_c(long long n, const double2* __restrict__ x, double* __restrict__ c) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) c[i] = x[i].x;
}

// |A_lin| |x| (+ |c| inv_dt on c rows): the cancellation floor scale (newton.py:62-72)
__global__ void k_abs_lin(DevParams P, const uint8_t* __restrict__ lab, const double2* __restrict__ X,
                          double inv_dt, double2* __restrict__ out) {
  int x, y, z, v;
  if (!vox_index(P, x, y, z, v)) return;
  uint8_t a = lab[v];
  if (z == P.nz - 1 && a == CC) { out[v] = make_double2(0.0, 0.0); return; }
  double2 xa = X[v];
  double ac = fabs(xa.x), ap = fabs(xa.y);
  double rc = 0.0, rp = 0.0;
  const double gM = P.t_plus * P.kappa * P.gF2;
  for (int d = 0; d < 6; ++d) {
    long long nb;
    int zb = z;
    if (d == 0) { if (x == 0) continue; nb = v - 1; }
    else if (d == 1) { if (x + 1 >= P.nx) continue; nb = v + 1; }
    else if (d == 2) { if (y == 0) continue; nb = v - P.nx; }
    else if (d == 3) { if (y + 1 >= P.ny) continue; nb = v + P.nx; }
    else if (d == 4) { if (z == 0) continue; nb = v - P.nxy; zb = z - 1; }
    else { if (z + 1 >= P.nz) continue; nb = v + P.nxy; zb = z + 1; }
    uint8_t b = lab[nb];
    uint8_t k = kind_of(a, b);
    bool gb = zb == P.nz - 1 && b == CC;
    double sa = P.sig[a], sb = P.sig[b];
    if (gb) {
      if (k == K_CONT || k == K_CONTACT) rp += 2.0 * sa * sb / (sa + sb) * P.gF2 * ap;
      continue;
    }
    double2 xb = X[nb];
    double bc = fabs(xb.x), bp = fabs(xb.y);
    if (k == K_CONT) {
      if (a == GR) {
        rc += P.d_gr * P.inv_h2 * (ac + bc);
        rp += P.sigma_gr * P.gF2 * (ap + bp);
      } else if (a == EL) {
        rc += P.d_el * P.inv_h2 * (ac + bc) + gM * (ap + bp);
        rp += P.kappa * P.gF2 * (ap + bp);
      } else {
        rp += P.sig[a] * P.gF2 * (ap + bp);
      }
    } else if (k == K_CONTACT) {
      rp += 2.0 * sa * sb / (sa + sb) * P.gF2 * (ap + bp);
    }
  }
  if (a == GR || a == EL) rc += ac * inv_dt;
  else rc = 0.0;
  out[v] = make_double2(rc, rp);
}

// positivity guard: partial minima of c / (-delta_c) over delta_c < 0
__global__ void k_pos_min(DevParams P, const uint8_t* __restrict__ lab, const double2* __restrict__ x,
                          const double2* __restrict__ d, double* __restrict__ part) {
  __shared__ double sh[32];
  double m = INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.nvox;
       i += (long long)gridDim.x * blockDim.x) {
    uint8_t a = lab[i];
    if (a != GR && a != EL) continue;
    double dc = d[i].x;
    if (dc < 0.0) m = fmin(m, x[i].x / -dc);
  }
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : INFINITY;
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_down_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) part[blockIdx.x] = m;
  }
}

// per plated slot: outflow (mol/s) through its stripping faces (timestepping.py:50-57),
// then n_new = max(0, n - dt*flux); part[] collects the clamped (negative) mass
__global__ void k_plated_update(DevParams P, long long n_pl, const int32_t* __restrict__ pl_vox,
                                const int32_t* __restrict__ if_rank, const int32_t* __restrict__ if_dir,
                                const int32_t* __restrict__ if_so, const int32_t* __restrict__ if_el,
                                const int8_t* __restrict__ if_kind, const double2* __restrict__ X,
                                const double* __restrict__ npl, double beta, double dt,
                                double face_area_over_F, double* __restrict__ npl_new,
                                double* __restrict__ clamp) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n_pl) return;
  int v = pl_vox[k];
  int rk = if_rank[v];
  double flux = 0.0;
  if (rk >= 0) {
    for (int d = 0; d < 6; ++d) {
      int f = if_dir[6LL * rk + d];
      if (f < 0 || if_kind[f] != IF_STRIP || if_so[f] != v) continue;
      double2 xs = X[v], xe = X[if_el[f]];
      double i = strip_current_dev(xe.x, xs.y, xe.y, npl[k], beta, P, nullptr, nullptr);
      flux += i * face_area_over_F;
    }
  }
  double nn = npl[k] - dt * flux;
  clamp[k] = nn < 0.0 ? -nn : 0.0;
  npl_new[k] = fmax(nn, 0.0);
}

__global__ void k_sum(long long n, const double* __restrict__ a, double* __restrict__ part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s += a[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}


// ---- device-resident Newton: scalar control kernels (state in ns[NS_*]) -------------
// block-wide fixed-order reduction (sum or min) of nb partials; valid in thread 0
template <bool MIN>
__device__ double ns_reduce(const double* part, int nb) {
  __shared__ double sh[32];
  double v = MIN ? INFINITY : 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v = MIN ? fmin(v, part[i]) : v + part[i];
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_down_sync(0xffffffffu, v, o);
    v = MIN ? fmin(v, u) : v + u;
  }
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : (MIN ? INFINITY : 0.0);
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_down_sync(0xffffffffu, v, o);
      v = MIN ? fmin(v, u) : v + u;
    }
  }
  __syncthreads();
  return v;
}

// norm of k_sumsq2 partials (fields separately, then masked; +inf if any is non-finite)
__global__ void k_ns_norm(int nb, const double* __restrict__ part, int mask, double scale, double* ns,
                          int slot) {
  const double c = ns_reduce<false>(part, nb);
  const double p = ns_reduce<false>(part + nb, nb);
  if (threadIdx.x != 0) return;
  double v;
  if (!isfinite(c) || !isfinite(p)) v = INFINITY;
  else v = sqrt((mask & 1 ? c : 0.0) + (mask & 2 ? p : 0.0));
  ns[slot] = scale * v;
}
// tolerance rule of newton.py: max(atol, rtol |F0|, floor); floor arrives in ns[NS_TOL]
__global__ void k_ns_init(double* ns, double atol, double rtol) {
  const double n0 = ns[NS_NORM0];
  ns[NS_IT] = 0.0;
  ns[NS_KITERS] = 0.0;
  ns[NS_NORM] = n0;
  ns[NS_WHY] = 0.0;
  if (!isfinite(n0)) { ns[NS_STATUS] = 2.0; ns[NS_WHY] = 1.0; return; }
  const double tol = fmax(fmax(atol, rtol * n0), ns[NS_TOL]);
  ns[NS_TOL] = tol;
  ns[NS_STATUS] = n0 <= tol ? 1.0 : 0.0;
}
__global__ void k_ns_newton_cond(const double* ns, cudaGraphConditionalHandle h, int max_iter) {
  cudaGraphSetConditional(h, (ns[NS_STATUS] == 0.0 && ns[NS_IT] < (double)max_iter) ? 1u : 0u);
}
__global__ void k_ns_rebuild_cond(const double* ns, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (ns[NS_IT] == 0.0 && ns[NS_REBUILD] != 0.0 && ns[NS_STATUS] == 0.0) ? 1u : 0u);
}
__global__ void k_ns_lintol(double* ns, double linear_rtol, double safety) {
  ns[NS_LINTOL] = fmin(0.1, fmax(linear_rtol, safety * ns[NS_TOL] / ns[NS_NORM]));
}
// positivity guard: alpha = min(1, 0.99 min_i c_i / -d_i) over the block minima
__global__ void k_ns_guard(int rb, const double* __restrict__ part, double* ns, cudaGraphConditionalHandle h) {
  const double lim = ns_reduce<true>(part, rb);
  if (threadIdx.x != 0) return;
  double alpha = 1.0;
  if (isfinite(lim)) alpha = fmin(alpha, 0.99 * lim);
  if (alpha <= 0.0 && ns[NS_STATUS] == 0.0) { ns[NS_STATUS] = 2.0; ns[NS_WHY] = 2.0; }
  ns[NS_ALPHA] = alpha;
  ns[NS_ACC] = 0.0;
  ns[NS_H] = 0.0;
  ns[NS_NTRY] = INFINITY;
  cudaGraphSetConditional(h, ns[NS_STATUS] == 0.0 ? 1u : 0u);
}
__global__ void k_ns_axpy(long long n, const double2* __restrict__ a, const double* __restrict__ ns,
                          const double2* __restrict__ b, double2* __restrict__ y) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double alpha = ns[NS_ALPHA];
  double2 u = a[i], w = b[i];
  y[i] = make_double2(u.x + alpha * w.x, u.y + alpha * w.y);
}
// backtracking (8 halvings): accept if finite and no worse than the current residual or
// already within tolerance; otherwise halve alpha and try again
__global__ void k_ns_ls(double* ns, cudaGraphConditionalHandle h) {
  const double nt = ns[NS_NTRY];
  if (isfinite(nt) && (nt <= ns[NS_NORM] || nt <= ns[NS_TOL])) ns[NS_ACC] = 1.0;
  else { ns[NS_ALPHA] *= 0.5; ns[NS_H] += 1.0; }
  cudaGraphSetConditional(h, (ns[NS_STATUS] == 0.0 && ns[NS_ACC] == 0.0 && ns[NS_H] <= 8.0) ? 1u : 0u);
}
__global__ void k_ns_lsfinal_cond(const double* ns, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, (ns[NS_STATUS] == 0.0 && ns[NS_ACC] == 0.0) ? 1u : 0u);
}
__global__ void k_ns_lsfinal_check(double* ns) {
  if (!isfinite(ns[NS_NTRY])) { ns[NS_STATUS] = 2.0; ns[NS_WHY] = 3.0; }
}
__global__ void k_ns_accept(double* ns) {
  if (ns[NS_STATUS] != 0.0) return;
  ns[NS_NORM] = ns[NS_NTRY];
  ns[NS_IT] += 1.0;
  if (ns[NS_NORM] <= ns[NS_TOL]) ns[NS_STATUS] = 1.0;
}
}  // namespace

// ------------------------------------------------------------------ workspace
Work& work(Operator& op) {
  if (!op.work) op.work = new Work(op.P.nvox);
  return *op.work;
}

Work::Work(long long nvox)
    : x(nvox), xt(nvox), r(nvox), rt(nvox), d(nvox), b(nvox), kr(nvox), khat(nvox), kp(nvox),
      kv(nvox), ks(nvox), kt(nvox), kph(nvox), ksh(nvox), cprev(nvox), part(8192), parth(8192) {
  // zeroed: the multigrid's c-block sweeps write only the planes that hold c rows; the c
  // entries of every other plane are zero in all Krylov vectors and stay so
  for (DBuf<double2>* b : {&x, &xt, &r, &rt, &d, &this->b, &kr, &khat, &kp, &kv, &ks, &kt, &kph, &ksh})
    HC_CUDA(cudaMemset(b->p, 0, (size_t)nvox * sizeof(double2)));
}

static int red_blocks(const Operator& op) {
  return (int)std::min<long long>(nblk(op.P.nvox), 4LL * op.n_sm);
}

static double host_sum(Operator& op, int nb, int off, cudaStream_t s) {
  Work& W = work(op);
  HC_CUDA(cudaMemcpyAsync(W.parth.data(), W.part.p + off, nb * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  for (int i = 0; i < nb; ++i) acc += W.parth[i];
  return acc;
}

double dot(Operator& op, const double2* a, const double2* b, cudaStream_t s) {
  int nb = red_blocks(op);
  k_dot2<<<nb, TPB, 0, s>>>(op.P.nvox, a, b, nullptr, nullptr, work(op).part.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  return host_sum(op, nb, 0, s);
}

void dot2(Operator& op, const double2* a, const double2* b, const double2* c, const double2* d,
          double& ab, double& cd, cudaStream_t s) {
  int nb = red_blocks(op);
  Work& W = work(op);
  k_dot2<<<nb, TPB, 0, s>>>(op.P.nvox, a, b, c, d, W.part.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaMemcpyAsync(W.parth.data(), W.part.p, 2 * nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  ab = cd = 0.0;
  for (int i = 0; i < nb; ++i) { ab += W.parth[i]; cd += W.parth[nb + i]; }
}

// returns sqrt of sum of squares over the fields in mask; +inf if any entry of
// EITHER field is non-finite (the reference raises NumericsError on any row)
double norm_checked(Operator& op, const double2* a, int mask, cudaStream_t s) {
  int nb = red_blocks(op);
  Work& W = work(op);
  k_sumsq2<<<nb, TPB, 0, s>>>(op.P.nvox, a, W.part.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaMemcpyAsync(W.parth.data(), W.part.p, 2 * nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  double c = 0.0, p = 0.0;
  for (int i = 0; i < nb; ++i) { c += W.parth[i]; p += W.parth[nb + i]; }
  if (!std::isfinite(c) || !std::isfinite(p)) return INFINITY;
  double acc = (mask & 1 ? c : 0.0) + (mask & 2 ? p : 0.0);
  return std::sqrt(acc);
}

// J-operator of the linear solve: mode 0 full J + mass, mode 1 phi block
static void apply_A(Operator& op, const double2* v, double2* out, double inv_dt, int mode,
                    cudaStream_t s) {
  jvp_grid(op, v, inv_dt, mode == 0 ? (1 | 4) : 8, out, s);
}

// Right-preconditioned BiCGStab on the grid layout; x starts at 0.
// Returns the number of iterations; throws NonConvergence on stall.
int bicgstab(Operator& op, const double2* b, double2* x, double inv_dt, int mode, double rtol,
             int maxit, cudaStream_t s) {
  Work& W = work(op);
  const long long n = op.P.nvox;
  const int nb = nblk(n);
  HC_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double2), s));
  double bnorm = std::sqrt(dot(op, b, b, s));
  if (bnorm == 0.0) return 0;
  if (!std::isfinite(bnorm)) throw Error(HC_ERR_NONCONVERGENCE, "non-finite Newton right-hand side");
  const double tol = rtol * bnorm;
  HC_CUDA(cudaMemcpyAsync(W.kr.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  HC_CUDA(cudaMemcpyAsync(W.khat.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  HC_CUDA(cudaMemsetAsync(W.kp.p, 0, n * sizeof(double2), s));
  HC_CUDA(cudaMemsetAsync(W.kv.p, 0, n * sizeof(double2), s));
  double rho = 1.0, alpha = 1.0, omega = 1.0;
  double rnorm = bnorm;
  for (int it = 1; it <= maxit; ++it) {
    double rho1 = dot(op, W.khat.p, W.kr.p, s);
    if (rho1 == 0.0 || !std::isfinite(rho1))
      throw Error(HC_ERR_NONCONVERGENCE, "iterative linear solver stalled (rho breakdown)");
    double beta = (rho1 / rho) * (alpha / omega);
    k_p_update<<<nb, TPB, 0, s>>>(n, beta, omega, W.kr.p, W.kv.p, W.kp.p); HC_COUNT();
    amg_apply(op, W.kp.p, W.kph.p, inv_dt, mode, s);
    apply_A(op, W.kph.p, W.kv.p, inv_dt, mode, s);
    double rv = dot(op, W.khat.p, W.kv.p, s);
    if (rv == 0.0 || !std::isfinite(rv))
      throw Error(HC_ERR_NONCONVERGENCE, "iterative linear solver stalled (alpha breakdown)");
    alpha = rho1 / rv;
    k_axpy<<<nb, TPB, 0, s>>>(n, W.kr.p, -alpha, W.kv.p, W.ks.p); HC_COUNT();
    double snorm = std::sqrt(dot(op, W.ks.p, W.ks.p, s));
    if (snorm <= tol) {
      k_axpy<<<nb, TPB, 0, s>>>(n, x, alpha, W.kph.p, x); HC_COUNT();
      HC_CHECK_LAUNCH();
      return it;
    }
    amg_apply(op, W.ks.p, W.ksh.p, inv_dt, mode, s);
    apply_A(op, W.ksh.p, W.kt.p, inv_dt, mode, s);
    double ts, tt;
    dot2(op, W.kt.p, W.ks.p, W.kt.p, W.kt.p, ts, tt, s);
    if (tt == 0.0 || !std::isfinite(tt))
      throw Error(HC_ERR_NONCONVERGENCE, "iterative linear solver stalled (omega breakdown)");
    omega = ts / tt;
    k_x_update<<<nb, TPB, 0, s>>>(n, alpha, W.kph.p, omega, W.ksh.p, x); HC_COUNT();
    k_axpy<<<nb, TPB, 0, s>>>(n, W.ks.p, -omega, W.kt.p, W.kr.p); HC_COUNT();
    HC_CHECK_LAUNCH();
    rnorm = std::sqrt(dot(op, W.kr.p, W.kr.p, s));
    if (op.krylov_log) fprintf(stderr, "krylov mode=%d it=%d relres=%.3e alpha=%.3e omega=%.3e\n", mode, it, rnorm / bnorm, alpha, omega);
    if (rnorm <= tol) return it;
    if (omega == 0.0)
      throw Error(HC_ERR_NONCONVERGENCE, "iterative linear solver stalled (omega = 0)");
    rho = rho1;
  }
  char msg[160];
  snprintf(msg, sizeof msg, "iterative linear solver stalled (info=%d, relres=%.3e)", maxit,
           rnorm / bnorm);
  throw Error(HC_ERR_NONCONVERGENCE, msg);
}

static double floor_norm(Operator& op, const double2* x, double inv_dt, cudaStream_t s) {
  Work& W = work(op);
  k_abs_lin<<<vox_grid(op.P), vox_block(), 0, s>>>(op.P, op.labels.p, x, inv_dt, W.rt.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  return 1e-13 * norm_checked(op, W.rt.p, 3, s);
}

static void ensure_amg(Operator& op) {
  if (!op.amg) op.amg = build_amg(op);
}

// ---- device-resident Newton solve -----------------------------------------------------
// The whole newton_solve of one implicit step (newton.py:86-168) as ONE CUDA graph: a
// WHILE node over Newton iterations whose body linearizes, rebuilds the multigrid values
// under an IF node, runs the BiCGStab WHILE loop, applies the positivity guard and the
// backtracking line search (another WHILE node) — every decision taken by one-thread
// kernels on device scalars.  The host launches the graph and reads the scalars once.
struct NewtonGraph {
  cudaGraphExec_t exec = nullptr;
  double dt = -1.0, mu = 0.0;
  const double* npl = nullptr;
  // work-buffer addresses captured into the graph (the host loops swap W.x/W.xt and
  // W.r/W.rt, so they are part of the key)
  const double2 *px = nullptr, *pxt = nullptr, *pr = nullptr, *prt = nullptr;
  hc_solver_config cfg{};
  DBuf<double> ns;
  double* ns_host = nullptr;
  unsigned long long per_iter_kernels = 0;
  ~NewtonGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (ns_host) cudaFreeHost(ns_host);
  }
};
void destroy_newton_graph(NewtonGraph* g) { delete g; }

static bool same_cfg(const hc_solver_config& a, const hc_solver_config& b) {
  return a.newton_rtol == b.newton_rtol && a.newton_atol == b.newton_atol &&
         a.newton_max_iter == b.newton_max_iter && a.krylov_max_iter == b.krylov_max_iter &&
         a.linear_rtol == b.linear_rtol && a.implicit_plated == b.implicit_plated &&
         a.linear_safety == b.linear_safety;
}

static void build_newton_graph(Operator& op, NewtonGraph& NG, const double* npl, double dt, double mu,
                               const hc_solver_config& cfg, cudaStream_t s) {
  Work& W = work(op);
  const long long n = op.P.nvox;
  const int nb = nblk(n);
  const int rb = red_blocks(op);
  const double inv_dt = 1.0 / dt;
  const double beta = cfg.implicit_plated ? dt * op.info.face_area / op.host_params.faraday : 0.0;
  const int parts = PART_LIN | PART_BV | PART_1C | PART_BND | PART_TIME;
  double* ns = NG.ns.p;
  cudaGraph_t outer;
  HC_CUDA(cudaGraphCreate(&outer, 0));
  // the multigrid's sparsified sweep patterns are decided at each block's first numeric
  // setup, which has to be an eager one: run it here when no solve has done so yet
  if (op.amg && !(op.amg->blk[0].sp_done && op.amg->blk[1].sp_done)) {
    linearize(op, W.x.p, npl, beta, s);
    amg_update(op, inv_dt, 3, s);
    op.amg->force = true;   // (the first solve still rebuilds the hierarchy at its own state)
  }
  const unsigned long long c0 = t_launch_count;
  op.capturing = true;
  try {
    GraphBuilder gb{s, outer, {}};
    auto norm_into = [&](const double2* v, int slot, double scale) {
      k_sumsq2<<<rb, TPB, 0, s>>>(n, v, W.part.p); HC_COUNT();
      k_ns_norm<<<1, 256, 0, s>>>(rb, W.part.p, 3, scale, ns, slot); HC_COUNT();
    };
    cudaGraphConditionalHandle hn = gb.handle(0);
    gb.capture([&] {
      residual_grid(op, W.x.p, npl, mu, beta, parts, W.cprev.p, inv_dt, W.r.p, s);
      norm_into(W.r.p, NS_NORM0, 1.0);
      k_abs_lin<<<vox_grid(op.P), vox_block(), 0, s>>>(op.P, op.labels.p, W.x.p, inv_dt, W.rt.p); HC_COUNT();
      norm_into(W.rt.p, NS_TOL, 1e-13);
      k_ns_init<<<1, 1, 0, s>>>(ns, cfg.newton_atol, cfg.newton_rtol); HC_COUNT();
      k_ns_newton_cond<<<1, 1, 0, s>>>(ns, hn, cfg.newton_max_iter); HC_COUNT();
    });
    GraphBuilder body{s, gb.cond(hn, cudaGraphCondTypeWhile), {}};
    cudaGraphConditionalHandle hr = body.handle(0);
    body.capture([&] {
      linearize(op, W.x.p, npl, beta, s);
      k_ns_rebuild_cond<<<1, 1, 0, s>>>(ns, hr); HC_COUNT();
    });
    {
      GraphBuilder rbld{s, body.cond(hr, cudaGraphCondTypeIf), {}};
      rbld.capture([&] { amg_update(op, inv_dt, 3, s); });
    }
    body.capture([&] {
      k_neg<<<nb, TPB, 0, s>>>(n, W.r.p, W.b.p); HC_COUNT();
      k_ns_lintol<<<1, 1, 0, s>>>(ns, cfg.linear_rtol, cfg.linear_safety); HC_COUNT();
    });
    krylov_append(op, body, W.b.p, W.d.p, inv_dt, 0, ns + NS_LINTOL, cfg.krylov_max_iter, ns);
    cudaGraphConditionalHandle hl = body.handle(0);
    body.capture([&] {
      k_pos_min<<<rb, TPB, 0, s>>>(op.P, op.labels.p, W.x.p, W.d.p, W.part.p); HC_COUNT();
      k_ns_guard<<<1, 256, 0, s>>>(rb, W.part.p, ns, hl); HC_COUNT();
    });
    auto trial = [&](GraphBuilder& b) {
      b.capture([&] {
        k_ns_axpy<<<nb, TPB, 0, s>>>(n, W.x.p, ns, W.d.p, W.xt.p); HC_COUNT();
        residual_grid(op, W.xt.p, npl, mu, beta, parts, W.cprev.p, inv_dt, W.rt.p, s);
        norm_into(W.rt.p, NS_NTRY, 1.0);
      });
    };
    {
      GraphBuilder ls{s, body.cond(hl, cudaGraphCondTypeWhile), {}};
      trial(ls);
      ls.capture([&] { k_ns_ls<<<1, 1, 0, s>>>(ns, hl); HC_COUNT(); });
    }
    cudaGraphConditionalHandle hf = body.handle(0);
    body.capture([&] { k_ns_lsfinal_cond<<<1, 1, 0, s>>>(ns, hf); HC_COUNT(); });
    {
      GraphBuilder fin{s, body.cond(hf, cudaGraphCondTypeIf), {}};
      trial(fin);
      fin.capture([&] { k_ns_lsfinal_check<<<1, 1, 0, s>>>(ns); HC_COUNT(); });
    }
    body.capture([&] {
      HC_CUDA(cudaMemcpyAsync(W.x.p, W.xt.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      HC_CUDA(cudaMemcpyAsync(W.r.p, W.rt.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      k_ns_accept<<<1, 1, 0, s>>>(ns); HC_COUNT();
      k_ns_newton_cond<<<1, 1, 0, s>>>(ns, hn, cfg.newton_max_iter); HC_COUNT();
    });
    op.capturing = false;
    NG.per_iter_kernels = t_launch_count - c0;
    uncount(t_launch_count - c0);
    if (NG.exec) cudaGraphExecDestroy(NG.exec);
    NG.exec = nullptr;
    HC_CUDA(cudaGraphInstantiate(&NG.exec, outer, 0));
    HC_CUDA(cudaGraphUpload(NG.exec, s));
  } catch (...) {
    op.capturing = false;
    uncount(t_launch_count - c0);
    cudaGraphDestroy(outer);
    cudaGetLastError();
    throw;
  }
  cudaGraphDestroy(outer);
  NG.dt = dt;
  NG.mu = mu;
  NG.npl = npl;
  NG.cfg = cfg;
  NG.px = W.x.p;
  NG.pxt = W.xt.p;
  NG.pr = W.r.p;
  NG.prt = W.rt.p;
}

// returns false if the device path is unavailable (the caller runs the host loop)
static bool newton_grid_dev(Operator& op, const double* npl, double dt, double mu,
                            const hc_solver_config& cfg, hc_newton_stats& st, cudaStream_t s) {
  Amg& A = *op.amg;
  if (!op.newton_dev || A.refresh || op.iter_out || op.trace_norms || op.src || !op.dev_krylov ||
      !op.krylov_while)
    return false;
  Work& W = work(op);
  if (!op.ng) {
    op.ng = new NewtonGraph();
    op.ng->ns.alloc(NS_N);
    HC_CUDA(cudaMallocHost(&op.ng->ns_host, NS_N * sizeof(double)));
  }
  NewtonGraph& NG = *op.ng;
  const double inv_dt = 1.0 / dt;
  if (!NG.exec || NG.dt != dt || NG.mu != mu || NG.npl != npl || !same_cfg(NG.cfg, cfg) ||
      NG.px != W.x.p || NG.pxt != W.xt.p || NG.pr != W.r.p || NG.prt != W.rt.p) {
    try {
      auto t0 = std::chrono::steady_clock::now();
      build_newton_graph(op, NG, npl, dt, mu, cfg, s);
      if (op.krylov_log)
        fprintf(stderr, "newton(dev): graph built in %.1f ms\n",
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    } catch (const Error& e) {
      if (op.krylov_log) fprintf(stderr, "newton: device graph unavailable (%s), host loop\n", e.what());
      op.newton_dev = false;
      return false;
    }
  }
  ++A.solves;
  const bool rebuild = A.force || A.solves % A.refresh_solves == 1 || A.refresh_solves == 1 ||
                       A.last_inv_dt != inv_dt;
  NG.ns_host[NS_REBUILD] = rebuild ? 1.0 : 0.0;
  HC_CUDA(cudaMemcpyAsync(NG.ns.p + NS_REBUILD, NG.ns_host + NS_REBUILD, sizeof(double),
                          cudaMemcpyHostToDevice, s));
  auto tl = std::chrono::steady_clock::now();
  HC_CUDA(cudaGraphLaunch(NG.exec, s));
  const double launch_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count();
  HC_CUDA(cudaMemcpyAsync(NG.ns_host, NG.ns.p, NS_N * sizeof(double), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  if (op.krylov_log)
    fprintf(stderr, "newton(dev): launch %.3f ms, launch+sync %.2f ms\n", launch_ms,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count());
  const double* h = NG.ns_host;
  if (op.krylov_log)
    fprintf(stderr, "newton(dev): dt=%g status=%g it=%g kiters=%g norm0=%.3e tol=%.3e norm=%.3e lintol=%.3e rebuild=%d why=%g\n",
            dt, h[NS_STATUS], h[NS_IT], h[NS_KITERS], h[NS_NORM0], h[NS_TOL], h[NS_NORM], h[NS_LINTOL],
            (int)rebuild, h[NS_WHY]);
  // a solve that converged at its initial residual ran no Newton iteration: like the host
  // loop it does not count towards the refresh period (and rebuilt nothing)
  const bool iterated = h[NS_IT] + (h[NS_STATUS] == 1.0 ? 0.0 : 1.0) > 0.0;
  if (!iterated) --A.solves;
  if (rebuild && iterated) {
    A.last_inv_dt = inv_dt;
    A.force = false;
  }
  count_graph_launch(NG.per_iter_kernels * (unsigned long long)std::max(1.0, h[NS_IT]));
  st.norm0 = h[NS_NORM0];
  st.tol = h[NS_TOL];
  st.n_iter = (int)h[NS_IT];
  st.norm_final = h[NS_NORM];
  st.krylov_iters += (int)h[NS_KITERS];
  if (h[NS_STATUS] == 1.0) return true;
  const int why = (int)h[NS_WHY];
  op.krylov_fail_stale = why >= 9 && !rebuild;
  char msg[200];
  if (why == 1)
    snprintf(msg, sizeof msg, "initial residual not evaluable: operator produced a non-finite value");
  else if (why == 2)
    snprintf(msg, sizeof msg, "positivity guard blocked the Newton step");
  else if (why == 3)
    snprintf(msg, sizeof msg, "residual not evaluable under damping");
  else if (why >= 9)
    snprintf(msg, sizeof msg, "iterative linear solver stalled (%s)", why == 9 ? "iteration budget" : "breakdown");
  else
    snprintf(msg, sizeof msg, "Newton did not reach tolerance %.3e in %d iterations (last residual %.3e)",
             h[NS_TOL], cfg.newton_max_iter, h[NS_NORM]);
  throw Error(HC_ERR_NONCONVERGENCE, msg);
}

// newton_solve (newton.py:86-168) on the grid layout.  W.x holds the guess on
// entry and the solution on exit; W.cprev holds c_prev per voxel.
void newton_grid(Operator& op, const double* npl, double dt, double mu, const hc_solver_config& cfg,
                 hc_newton_stats& st, cudaStream_t s) {
  if (!(dt > 0)) throw Error(HC_ERR_ARGUMENT, "dt must be positive");
  ensure_amg(op);
  if (newton_grid_dev(op, npl, dt, mu, cfg, st, s)) return;
  Work& W = work(op);
  const long long n = op.P.nvox;
  const int nb = nblk(n);
  const double inv_dt = 1.0 / dt;
  const double beta = cfg.implicit_plated ? dt * op.info.face_area / op.host_params.faraday : 0.0;
  const int parts = PART_LIN | PART_BV | PART_1C | PART_BND | PART_TIME;
  // residual of newton.py:101-106: m (x - x_prev)/dt + A(x; mu) (+ source)
  auto residual = [&](const double2* xg, double2* out) {
    residual_grid(op, xg, npl, mu, beta, parts, W.cprev.p, inv_dt, out, s);
    if (op.src) { k_axpy<<<nb, TPB, 0, s>>>(n, out, 1.0, op.src, out); HC_COUNT(); }
  };
  op.iter_count = 0;
  op.norm_log.clear();
  residual(W.x.p, W.r.p);
  double norm0 = norm_checked(op, W.r.p, 3, s);
  if (!std::isfinite(norm0))
    throw Error(HC_ERR_NONCONVERGENCE, "initial residual not evaluable: operator produced a non-finite value");
  double tol = std::max({cfg.newton_atol, cfg.newton_rtol * norm0, floor_norm(op, W.x.p, inv_dt, s)});
  st.norm0 = norm0;
  st.tol = tol;
  st.n_iter = 0;
  st.norm_final = norm0;
  if (op.trace_norms) op.norm_log.push_back(norm0);
  if (norm0 <= tol) return;
  double norm = norm0;
  bool rebuilt = false;
  for (int it = 1; it <= cfg.newton_max_iter; ++it) {
    linearize(op, W.x.p, npl, beta, s);
    // the preconditioner is rebuilt at the first Newton iteration of every solve; later
    // iterations reuse it (the Krylov solver sees the exact current Jacobian)
    {
      Amg& A = *op.amg;
      bool first = it == 1;
      if (first) ++A.solves;
      // the Galerkin hierarchy is rebuilt for the first Newton iteration of every
      // refresh_solves-th solve (and always when dt changed); Krylov always sees the
      // exact current Jacobian, the preconditioner may lag
      bool rebuild = A.refresh || (first && (A.force || A.solves % A.refresh_solves == 1 ||
                                             A.refresh_solves == 1 || A.last_inv_dt != inv_dt));
      if (rebuild) {
        amg_update(op, inv_dt, 3, s);
        A.last_inv_dt = inv_dt;
        A.force = false;
        rebuilt = true;
      }
    }
    k_neg<<<nb, TPB, 0, s>>>(n, W.r.p, W.b.p); HC_COUNT();
    const double lin_tol = std::min(0.1, std::max(cfg.linear_rtol, cfg.linear_safety * tol / norm));
    try {
      st.krylov_iters += op.dev_krylov
          ? bicgstab_dev(op, W.b.p, W.d.p, inv_dt, 0, lin_tol, cfg.krylov_max_iter, s)
          : bicgstab(op, W.b.p, W.d.p, inv_dt, 0, lin_tol, cfg.krylov_max_iter, s);
    } catch (const Error& e) {
      op.krylov_fail_stale = e.code == HC_ERR_NONCONVERGENCE && !rebuilt;
      throw;
    }
    // positivity guard on the concentration block
    double alpha = 1.0;
    {
      int rb = red_blocks(op);
      k_pos_min<<<rb, TPB, 0, s>>>(op.P, op.labels.p, W.x.p, W.d.p, W.part.p); HC_COUNT();
      HC_CHECK_LAUNCH();
      HC_CUDA(cudaMemcpyAsync(W.parth.data(), W.part.p, rb * sizeof(double), cudaMemcpyDeviceToHost, s));
      HC_CUDA(cudaStreamSynchronize(s));
      double lim = INFINITY;
      for (int i = 0; i < rb; ++i) lim = std::min(lim, W.parth[i]);
      if (std::isfinite(lim)) alpha = std::min(alpha, 0.99 * lim);
    }
    if (alpha <= 0.0) throw Error(HC_ERR_NONCONVERGENCE, "positivity guard blocked the Newton step");
    bool accepted = false;
    double norm_try = INFINITY;
    for (int h = 0; h <= 8; ++h) {
      k_axpy<<<nb, TPB, 0, s>>>(n, W.x.p, alpha, W.d.p, W.xt.p); HC_COUNT();
      residual(W.xt.p, W.rt.p);
      norm_try = norm_checked(op, W.rt.p, 3, s);
      if (std::isfinite(norm_try) && (norm_try <= norm || norm_try <= tol)) { accepted = true; break; }
      alpha *= 0.5;
    }
    if (!accepted) {
      k_axpy<<<nb, TPB, 0, s>>>(n, W.x.p, alpha, W.d.p, W.xt.p); HC_COUNT();
      residual(W.xt.p, W.rt.p);
      norm_try = norm_checked(op, W.rt.p, 3, s);
      if (!std::isfinite(norm_try))
        throw Error(HC_ERR_NONCONVERGENCE, "residual not evaluable under damping");
    }
    std::swap(W.x.p, W.xt.p);
    std::swap(W.r.p, W.rt.p);
    norm = norm_try;
    st.n_iter = it;
    st.norm_final = norm;
    if (op.trace_norms) op.norm_log.push_back(norm);
    if (op.iter_out && op.iter_count < op.iter_max)
      gather_packed(op, W.x.p, op.iter_out + (long long)op.iter_count * (op.info.n_c + op.info.n_p), s);
    ++op.iter_count;
    if (norm <= tol) return;
  }
  char msg[200];
  snprintf(msg, sizeof msg, "Newton did not reach tolerance %.3e in %d iterations (last residual %.3e)",
           tol, cfg.newton_max_iter, norm);
  throw Error(HC_ERR_NONCONVERGENCE, msg);
}

// solve_initial_potential (newton.py:171-206): W.x in/out.
void initial_potential_grid(Operator& op, const double* npl, double mu, const hc_solver_config& cfg,
                            hc_newton_stats& st, cudaStream_t s) {
  ensure_amg(op);
  Work& W = work(op);
  const long long n = op.P.nvox;
  const int nb = nblk(n);
  const int parts = PART_LIN | PART_BV | PART_1C | PART_BND;
  residual_grid(op, W.x.p, npl, mu, 0.0, parts, nullptr, 0.0, W.r.p, s);
  double norm0 = norm_checked(op, W.r.p, 2, s);
  double tol = std::max({cfg.newton_atol, cfg.newton_rtol * norm0, floor_norm(op, W.x.p, 0.0, s)});
  st.norm0 = norm0;
  st.tol = tol;
  st.n_iter = 0;
  st.norm_final = norm0;
  if (norm0 <= tol) return;
  double norm = norm0;
  for (int it = 1; it <= cfg.newton_max_iter; ++it) {
    linearize(op, W.x.p, npl, 0.0, s);
    if (it == 1 || op.amg->refresh) amg_update(op, 0.0, 2, s);
    k_neg<<<nb, TPB, 0, s>>>(n, W.r.p, W.b.p); HC_COUNT();
    k_zero_c<<<nb, TPB, 0, s>>>(n, W.b.p); HC_COUNT();
    const double lin_tol = std::min(0.1, std::max(cfg.linear_rtol, cfg.linear_safety * tol / norm));
    st.krylov_iters += op.dev_krylov
        ? bicgstab_dev(op, W.b.p, W.d.p, 0.0, 1, lin_tol, cfg.krylov_max_iter, s)
        : bicgstab(op, W.b.p, W.d.p, 0.0, 1, lin_tol, cfg.krylov_max_iter, s);
    double alpha = 1.0, norm_try = INFINITY;
    for (int h = 0; h <= 8; ++h) {
      k_axpy<<<nb, TPB, 0, s>>>(n, W.x.p, alpha, W.d.p, W.xt.p); HC_COUNT();
      residual_grid(op, W.xt.p, npl, mu, 0.0, parts, nullptr, 0.0, W.rt.p, s);
      norm_try = norm_checked(op, W.rt.p, 2, s);
      if (std::isfinite(norm_try) && (norm_try <= norm || norm_try <= tol)) break;
      alpha *= 0.5;
    }
    std::swap(W.x.p, W.xt.p);
    std::swap(W.r.p, W.rt.p);
    norm = norm_try;
    st.n_iter = it;
    st.norm_final = norm;
    if (norm <= tol) return;
  }
  char msg[160];
  snprintf(msg, sizeof msg, "stationary potential solve stalled at residual %.3e", norm);
  throw Error(HC_ERR_NONCONVERGENCE, msg);
}

// step (timestepping.py:64-106) on the grid layout: W.x holds the state on
// entry (also x_prev) and the accepted state on exit; npl updated in place.
void step_grid(Operator& op, double* npl, double dt_suggest, double mu, const hc_solver_config& cfg,
               hc_newton_stats& st, cudaStream_t s) {
  Work& W = work(op);
  const long long n = op.P.nvox;
  double dt = std::min(dt_suggest, cfg.dt_max);
  int retries = 0;
  k_extract_c<<<nblk(n), TPB, 0, s>>>(n, W.x.p, W.cprev.p); HC_COUNT();
  DBuf<double2>& xprev = W.xprev_store;
  if (!xprev.p) xprev.alloc(n);
  HC_CUDA(cudaMemcpyAsync(xprev.p, W.x.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  st.krylov_iters = 0;
  bool stale_retry = false;
  while (true) {
    try {
      op.krylov_fail_stale = false;
      newton_grid(op, npl, dt, mu, cfg, st, s);
    } catch (const Error& e) {
      if (e.code != HC_ERR_NONCONVERGENCE) throw;
      if (op.krylov_fail_stale && !stale_retry) {
        // the Krylov solve failed on a lagged multigrid hierarchy: rebuild it and retry the
        // same dt (the reference's direct solve never fails here, so this is not a retry of
        // the step-size control)
        stale_retry = true;
        op.amg->force = true;
        HC_CUDA(cudaMemcpyAsync(W.x.p, xprev.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        continue;
      }
      stale_retry = true;   // a fresh hierarchy failed too: shrink dt as the reference does
      if (dt <= cfg.dt_min * (1.0 + 1e-12)) {
        char msg[256];
        snprintf(msg, sizeof msg, "time step underflow (dt=%.3e): %s", dt, e.what());
        throw Error(HC_ERR_SIMULATION, msg);
      }
      dt = std::max(dt * cfg.shrink_factor, cfg.dt_min);
      retries++;
      HC_CUDA(cudaMemcpyAsync(W.x.p, xprev.p, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
      continue;
    }
    break;
  }
  double clamped = 0.0;
  long long npls = op.info.n_plated;
  if (npls) {
    const double beta = cfg.implicit_plated ? dt * op.info.face_area / op.host_params.faraday : 0.0;
    DBuf<double>& tmp = W.npl_tmp;
    if (tmp.n < (size_t)(2 * npls)) tmp.alloc(2 * npls);
    k_plated_update<<<nblk(npls), TPB, 0, s>>>(op.P, npls, op.plated_vox.p, op.if_rank.p, op.if_dir.p,
                                               op.if_solid.p, op.if_el.p, op.if_kind.p, W.x.p, npl,
                                               beta, dt, op.info.face_area / op.host_params.faraday,
                                               tmp.p, tmp.p + npls); HC_COUNT();
    HC_CUDA(cudaMemcpyAsync(npl, tmp.p, npls * sizeof(double), cudaMemcpyDeviceToDevice, s));
    int rb = (int)std::min<long long>(nblk(npls), 1024);
    k_sum<<<rb, TPB, 0, s>>>(npls, tmp.p + npls, W.part.p); HC_COUNT();
    HC_CHECK_LAUNCH();
    clamped = host_sum(op, rb, 0, s);
  }
  st.dt_used = dt;
  st.retries = retries;
  st.clamped_loss = clamped;
  st.dt_next = st.n_iter <= cfg.easy_iter_threshold ? std::min(dt * cfg.grow_factor, cfg.dt_max) : dt;
}

}  // namespace hc
