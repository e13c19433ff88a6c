// Device-resident BiCGStab: scalars live in device memory, dot products are fused
// into the vector-update kernels as per-block partials that the kernel's last block
// finalizes (ticket pattern, fixed summation order), and one iteration is a single
// CUDA graph; the whole solve is one graph with a WHILE conditional node (fallback:
// batches of iteration graphs with one status read per batch).  Kernels become no-ops
// once the device has declared convergence.
//
// Algorithm and breakdown/stall semantics: right-preconditioned BiCGStab as in
// bicgstab() (hc_solver.cu), which replaces the reference's direct / ILU-LGMRES
// solve (fvm/newton.py:75-83).
#include <cmath>

#include "hc_amg.cuh"
#include "hc_solver.cuh"

namespace hc {

namespace {
constexpr int TPB = 256;
// device scalar slots
enum { S_RHO, S_ALPHA, S_OMEGA, S_RHO1, S_BETA, S_TOL2, S_RN2, S_SN2, S_DONE, S_ITERS, S_ERR,
       S_EARLY, S_RV, S_TS, S_TT, S_NSLOT };

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// block-reduce up to two sums into part[blockIdx.x] and part[gridDim.x + blockIdx.x]
__device__ __forceinline__ void block_part2(double s1, double s2, double* part) {
  __shared__ double sh[2][32];
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = s1; sh[1][w] = s2; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s1 = l < nw ? sh[0][l] : 0.0;
    s2 = l < nw ? sh[1][l] : 0.0;
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (l == 0) { part[blockIdx.x] = s1; part[gridDim.x + blockIdx.x] = s2; }
  }
}

// block-wide sum of nb partials in a fixed order (deterministic); result valid in thread 0
__device__ __forceinline__ double fin_sum_block(const double* part, int nb) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += __ldcg(part + i);   // other blocks' partials
  s = warp_sum(s);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = s;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
    t = warp_sum(t);
  }
  return t;
}

// fixed-order sum of n partials, result in every thread (every block computes the same)
__device__ __forceinline__ double block_sum_all(const double* part, int n) {
  __shared__ double sh[33];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += __ldcg(part + i);
  s = warp_sum(s);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = s;
  __syncthreads();
  if (w == 0) {
    double t = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

__device__ void finish_in_last_block(int what, const double* part, double* ks, unsigned* ticket);

// blocks per SM of the Krylov vector kernels (grid-stride loops over the voxels);
// enough blocks that every thread has only a few elements in flight
static int krylov_blocks_per_sm() {
  static int b = 0;
  if (!b) {
    const char* e = getenv("HC_KRYLOV_BPSM");
    b = std::max(1, e ? atoi(e) : 4);
  }
  return b;
}

__global__ void k_dev_dot2(long long n, double* ks, const double2* __restrict__ a,
                           const double2* __restrict__ b, const double2* __restrict__ c,
                           const double2* __restrict__ d, double* __restrict__ part, int what,
                           unsigned* ticket) {
  pdl_wait();
  if (ks[S_DONE] != 0.0) return;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll 2
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 x = a[i], y = b[i];
    s1 += x.x * y.x + x.y * y.y;
    if (c) {
      double2 u = c[i], w = d[i];
      s2 += u.x * w.x + u.y * w.y;
    }
  }
  block_part2(s1, s2, part);
  if (what >= 0) finish_in_last_block(what, part, ks, ticket);
}

// 0: beta  1: alpha  2: s-norm  3: omega  4: r-norm / next rho   (one block of 256)
__device__ void scalar_step(int what, int nb, const double* part, double* ks) {
  double s1 = 0.0, s2 = 0.0;
  if (what >= 1) s1 = fin_sum_block(part, nb);
  if (what >= 3) s2 = fin_sum_block(part + nb, nb);
  if (threadIdx.x != 0) return;
  if (what == 0) {
    double rho1 = ks[S_RHO1];
    if (rho1 == 0.0 || !isfinite(rho1)) { ks[S_ERR] = 1; ks[S_DONE] = 1; return; }
    ks[S_BETA] = (rho1 / ks[S_RHO]) * (ks[S_ALPHA] / ks[S_OMEGA]);
  } else if (what == 1) {
    double rv = s1;
    if (rv == 0.0 || !isfinite(rv)) { ks[S_ERR] = 2; ks[S_DONE] = 1; return; }
    ks[S_ALPHA] = ks[S_RHO1] / rv;
  } else if (what == 2) {
    ks[S_SN2] = s1;
    if (s1 <= ks[S_TOL2]) ks[S_EARLY] = 1;
  } else if (what == 3) {
    if (ks[S_EARLY] != 0.0) { ks[S_OMEGA] = 0.0; return; }
    double ts = s1, tt = s2;
    if (tt == 0.0 || !isfinite(tt)) { ks[S_ERR] = 3; ks[S_DONE] = 1; return; }
    ks[S_OMEGA] = ts / tt;
  } else {
    double rn2 = s1, rr = s2;
    ks[S_RN2] = rn2;
    ks[S_ITERS] += 1.0;
    ks[S_RHO] = ks[S_RHO1];
    ks[S_RHO1] = rr;
    if (ks[S_EARLY] != 0.0 || rn2 <= ks[S_TOL2]) { ks[S_DONE] = 1; return; }
    if (ks[S_OMEGA] == 0.0) { ks[S_ERR] = 4; ks[S_DONE] = 1; }
  }
}

__global__ void k_dev_scalar(int what, int nb, const double* __restrict__ part, double* ks) {
  pdl_wait();
  if (ks[S_DONE] != 0.0) return;
  scalar_step(what, nb, part, ks);
}

// The last block of a partial-producing kernel finalizes the scalar step itself
// (threadfence + ticket): one launch per reduction instead of two.  The partials are
// still summed in a fixed order, so the result is unchanged.
__device__ void finish_in_last_block(int what, const double* part, double* ks, unsigned* ticket) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  scalar_step(what, gridDim.x, part, ks);
  if (threadIdx.x == 0) *ticket = 0u;
}

// (rc, rp non-null: also the preconditioner's scalar right-hand sides T p_c, p_phi)
struct SplitOut {
  const uint8_t* lab;
  double tp;
  double* rc;
  double* rp;
  __device__ __forceinline__ void put(long long i, double2 a) const {
    if (!rc) return;
    rc[i] = lab[i] == EL ? a.x - tp * a.y : a.x;
    rp[i] = a.y;
  }
};

__global__ void k_dev_p(long long n, double* ks, const double2* __restrict__ r,
                        const double2* __restrict__ v, double2* __restrict__ p, SplitOut so) {
  pdl_wait();
  if (ks[S_DONE] != 0.0) return;
  // beta = (rho1 / rho) (alpha / omega), formerly k_dev_scalar(0): every thread derives it
  const double rho1 = ks[S_RHO1];
  const double beta = (rho1 / ks[S_RHO]) * (ks[S_ALPHA] / ks[S_OMEGA]), omega = ks[S_OMEGA];
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i == 0 && (rho1 == 0.0 || !isfinite(rho1))) { ks[S_ERR] = 1; ks[S_DONE] = 1; }
  if (i >= n) return;
  double2 pi = p[i], ri = r[i], vi = v[i];
  const double2 pn = make_double2(ri.x + beta * (pi.x - omega * vi.x), ri.y + beta * (pi.y - omega * vi.y));
  p[i] = pn;
  so.put(i, pn);
}

// s = r - alpha v, partial ||s||^2
__global__ void k_dev_s(long long n, double* ks, const double2* __restrict__ r,
                        const double2* __restrict__ v, double2* __restrict__ s,
                        double* __restrict__ part, unsigned* ticket, SplitOut so,
                        const double* __restrict__ jpart, int jnb) {
  pdl_wait();
  if (ks[S_DONE] != 0.0) return;
  double alpha;
  if (jnb > 0) {   // <rhat, v> from the J v epilogue's partials, summed by every block alike
    const double rv = block_sum_all(jpart, jnb);
    if (rv == 0.0 || !isfinite(rv)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) { ks[S_ERR] = 2; ks[S_DONE] = 1; }
      return;
    }
    alpha = ks[S_RHO1] / rv;
    if (blockIdx.x == 0 && threadIdx.x == 0) ks[S_ALPHA] = alpha;
  } else {
    alpha = ks[S_ALPHA];
  }
  double acc = 0.0;
#pragma unroll 2
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 ri = r[i], vi = v[i];
    double2 si = make_double2(ri.x - alpha * vi.x, ri.y - alpha * vi.y);
    s[i] = si;
    so.put(i, si);
    acc += si.x * si.x + si.y * si.y;
  }
  block_part2(acc, 0.0, part);
  finish_in_last_block(2, part, ks, ticket);
}

// x += alpha phat + omega shat; r = s - omega t; partials ||r||^2 and <rhat, r>
__global__ void k_dev_xr(long long n, double* ks, const double2* __restrict__ ph,
                         const double2* __restrict__ sh, const double2* __restrict__ s,
                         const double2* __restrict__ t, const double2* __restrict__ rhat,
                         double2* __restrict__ x, double2* __restrict__ r, double* __restrict__ part,
                         unsigned* ticket, const double* __restrict__ jpart, int jnb) {
  pdl_wait();
  if (ks[S_DONE] != 0.0) return;
  const double alpha = ks[S_ALPHA];
  double omega;
  if (jnb > 0) {   // omega = <t, s> / <t, t> from the J v epilogue's partials (scalar_step 3)
    if (ks[S_EARLY] != 0.0) {
      omega = 0.0;
    } else {
      const double ts = block_sum_all(jpart, jnb), tt = block_sum_all(jpart + jnb, jnb);
      if (tt == 0.0 || !isfinite(tt)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { ks[S_ERR] = 3; ks[S_DONE] = 1; }
        return;
      }
      omega = ts / tt;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ks[S_OMEGA] = omega;
  } else {
    omega = ks[S_OMEGA];
  }
  double a1 = 0.0, a2 = 0.0;
#pragma unroll 2
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 xi = x[i], pi = ph[i], si = sh[i], s0 = s[i], ti = t[i], h = rhat[i];
    x[i] = make_double2(xi.x + alpha * pi.x + omega * si.x, xi.y + alpha * pi.y + omega * si.y);
    double2 ri = make_double2(s0.x - omega * ti.x, s0.y - omega * ti.y);
    r[i] = ri;
    a1 += ri.x * ri.x + ri.y * ri.y;
    a2 += h.x * ri.x + h.y * ri.y;
  }
  block_part2(a1, a2, part);
  finish_in_last_block(4, part, ks, ticket);
}

// WHILE-node condition of the device-resident loop: continue while not converged / broken
// down and under the iteration budget
__global__ void k_dev_cond(const double* __restrict__ ks, cudaGraphConditionalHandle h, int maxit) {
  pdl_wait();
  cudaGraphSetConditional(h, (ks[S_DONE] == 0.0 && ks[S_ITERS] < (double)maxit) ? 1u : 0u);
}

// k_dev_init with the relative tolerance read from device memory (device Newton)
__global__ void k_dev_init_dev(int nb, const double* __restrict__ part, double* ks,
                               const double* __restrict__ rtol) {
  pdl_wait();
  double b2 = fin_sum_block(part, nb);
  if (threadIdx.x != 0) return;
  const double t = *rtol;
  for (int i = 0; i < S_NSLOT; ++i) ks[i] = 0.0;
  ks[S_RHO] = ks[S_ALPHA] = ks[S_OMEGA] = 1.0;
  ks[S_RHO1] = b2;
  ks[S_TOL2] = t * t * b2;
  if (b2 == 0.0) ks[S_DONE] = 1;
}

// after a device-resident solve: breakdown or budget exhaustion fails the Newton step
__global__ void k_dev_check(const double* __restrict__ ks, int maxit, double* ns) {
  pdl_wait();
  ns[NS_KITERS] += ks[S_ITERS];
  if (ks[S_ERR] != 0.0 || ks[S_DONE] == 0.0) {
    ns[NS_STATUS] = 2.0;
    ns[NS_WHY] = ks[S_ERR] != 0.0 ? 10.0 + ks[S_ERR] : 9.0;
  }
}

__global__ void k_dev_init(int nb, const double* __restrict__ part, double* ks, double tol2) {
  pdl_wait();
  double b2 = fin_sum_block(part, nb);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S_NSLOT; ++i) ks[i] = 0.0;
  ks[S_RHO] = ks[S_ALPHA] = ks[S_OMEGA] = 1.0;
  ks[S_RHO1] = b2;
  ks[S_TOL2] = tol2 * b2;
  if (b2 == 0.0) ks[S_DONE] = 1;
}
}  // namespace

struct KrylovGraphs {
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // per mode: one iteration
  cudaGraphExec_t loop[2] = {nullptr, nullptr};  // per mode: WHILE node around the iteration
  int loop_maxit[2] = {-1, -1};
  double inv_dt[2] = {-1.0, -1.0};
  unsigned long long n_kernels[2] = {0, 0};
  double2* x_ptr[2] = {nullptr, nullptr};
  DBuf<double> ks, part;
  DBuf<double> jpart;      // per-CTA dot partials of the two J v launches (fused epilogue)
  DBuf<unsigned> ticket;   // last-block ticket of the fused reductions (self-resetting)
  double* ks_host = nullptr;
  ~KrylovGraphs() {
    for (auto e : exec) if (e) cudaGraphExecDestroy(e);
    for (auto e : loop) if (e) cudaGraphExecDestroy(e);
    if (ks_host) cudaFreeHost(ks_host);
  }
};

void destroy_krylov_graphs(KrylovGraphs* g) { delete g; }

static void apply_A_dev(Operator& op, const double2* v, double2* out, double inv_dt, int mode,
                        cudaStream_t s) {
  jvp_grid(op, v, inv_dt, mode == 0 ? (1 | 4) : 8, out, s);
}

// upper bound on the CTAs of one TMA J v launch (one per tile column and plane)
static long long jpart_cap(const Operator& op) {
  return (long long)((op.P.nx + VX - 1) / VX) * ((op.P.ny + VY - 1) / VY) * op.P.nz;
}

// one BiCGStab iteration (captured into the iteration / WHILE-body graphs).  On the TMA
// path the two reductions after J v (<rhat, v>; <t, s>, <t, t>) come out of the J v
// kernel's epilogue as per-CTA partials and the next vector kernel sums them, so
// there is no separate reduction launch.
static void bicgstab_iteration(Operator& op, Work& W, KrylovGraphs& G, const SplitOut& so, double2* x,
                               double inv_dt, int mode, int nb, long long n, cudaStream_t s) {
  double* ks = G.ks.p;
  double* part = G.part.p;
  unsigned* tk = G.ticket.p;
  const int flags = mode == 0 ? (1 | 4) : 8;
  const long long jcap = jpart_cap(op);
  double* jp1 = G.jpart.p;
  double* jp2 = G.jpart.p + jcap;
  launch(k_dev_p, (int)((n + TPB - 1) / TPB), TPB, 0, s, n, ks, W.kr.p, W.kv.p, W.kp.p, so); HC_COUNT();
  amg_apply(op, W.kp.p, W.kph.p, inv_dt, mode, s, true);
  int j1 = jvp_grid_dot(op, W.kph.p, inv_dt, flags, W.kv.p, W.khat.p, jp1, 0, s);
  if (!j1) {
    apply_A_dev(op, W.kph.p, W.kv.p, inv_dt, mode, s);
    launch(k_dev_dot2, nb, TPB, 0, s, n, ks, W.khat.p, W.kv.p, nullptr, nullptr, part, 1, tk); HC_COUNT();
  }
  launch(k_dev_s, nb, TPB, 0, s, n, ks, W.kr.p, W.kv.p, W.ks.p, part, tk, so, (const double*)jp1, j1);
  HC_COUNT();
  amg_apply(op, W.ks.p, W.ksh.p, inv_dt, mode, s, true);
  int j2 = jvp_grid_dot(op, W.ksh.p, inv_dt, flags, W.kt.p, W.ks.p, jp2, 1, s);
  if (!j2) {
    apply_A_dev(op, W.ksh.p, W.kt.p, inv_dt, mode, s);
    launch(k_dev_dot2, nb, TPB, 0, s, n, ks, W.kt.p, W.ks.p, W.kt.p, W.kt.p, part, 3, tk); HC_COUNT();
  }
  launch(k_dev_xr, nb, TPB, 0, s, n, ks, W.kph.p, W.ksh.p, W.ks.p, W.kt.p, W.khat.p, x, W.kr.p, part, tk,
         (const double*)jp2, j2);
  HC_COUNT();
}

int bicgstab_dev(Operator& op, const double2* b, double2* x, double inv_dt, int mode, double rtol,
                 int maxit, cudaStream_t s) {
  Work& W = work(op);
  if (!op.kg) op.kg = new KrylovGraphs();
  KrylovGraphs& G = *op.kg;
  const long long n = op.P.nvox;
  const int nb = (int)std::min<long long>((n + TPB - 1) / TPB, (long long)krylov_blocks_per_sm() * op.n_sm);
  if (!G.ks.p) {
    G.ks.alloc(S_NSLOT);
    G.part.alloc(4 * nb + 8);
    G.jpart.alloc(3 * jpart_cap(op));
    G.ticket.alloc(1);
    HC_CUDA(cudaMemset(G.ticket.p, 0, sizeof(unsigned)));
    HC_CUDA(cudaMallocHost(&G.ks_host, S_NSLOT * sizeof(double)));
  }
  // init: x = 0, r = rhat = b, p = v = 0
  HC_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double2), s));
  HC_CUDA(cudaMemcpyAsync(W.kr.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  HC_CUDA(cudaMemcpyAsync(W.khat.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  HC_CUDA(cudaMemsetAsync(W.kp.p, 0, n * sizeof(double2), s));
  HC_CUDA(cudaMemsetAsync(W.kv.p, 0, n * sizeof(double2), s));
  HC_CUDA(cudaMemsetAsync(G.ks.p, 0, S_NSLOT * sizeof(double), s));
  launch(k_dev_dot2, nb, TPB, 0, s, n, G.ks.p, b, b, nullptr, nullptr, G.part.p, -1, G.ticket.p); HC_COUNT();
  launch(k_dev_init, 1, 256, 0, s, nb, G.part.p, G.ks.p, rtol * rtol); HC_COUNT();
  // the body of one BiCGStab iteration (captured, never run eagerly)
  const SplitOut so{op.labels.p, op.P.t_plus, op.amg->rs[0].p, op.amg->rs[1].p};
  auto iteration = [&]() { bicgstab_iteration(op, W, G, so, x, inv_dt, mode, nb, n, s); };
  const bool rebuild = !G.exec[mode] || G.inv_dt[mode] != inv_dt;
  if (rebuild) {
    if (G.exec[mode]) cudaGraphExecDestroy(G.exec[mode]);
    if (G.loop[mode]) cudaGraphExecDestroy(G.loop[mode]);
    G.exec[mode] = G.loop[mode] = nullptr;
    unsigned long long c0 = t_launch_count;
    cudaGraph_t graph;
    op.capturing = true;
    HC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    iteration();
    HC_CUDA(cudaStreamEndCapture(s, &graph));
    op.capturing = false;
    G.n_kernels[mode] = t_launch_count - c0;
    uncount(G.n_kernels[mode]);
    HC_CUDA(cudaGraphInstantiate(&G.exec[mode], graph, 0));
    HC_CUDA(cudaGraphDestroy(graph));
    G.inv_dt[mode] = inv_dt;
    G.x_ptr[mode] = x;
  }
  if (op.krylov_while && (rebuild || G.loop_maxit[mode] != maxit)) {
    // the whole solve as ONE graph: a WHILE conditional node whose body is one iteration
    // and whose condition a device kernel sets from the convergence flag — no host
    // round trip until the solve is finished
    if (G.loop[mode]) cudaGraphExecDestroy(G.loop[mode]);
    G.loop[mode] = nullptr;
    cudaGraph_t outer = nullptr;
    bool ok = cudaGraphCreate(&outer, 0) == cudaSuccess;
    cudaGraphConditionalHandle h = 0;
    ok = ok && cudaGraphConditionalHandleCreate(&h, outer, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    ok = ok && cudaGraphAddNode(&node, outer, nullptr, 0, &np) == cudaSuccess;
    if (ok) {
      cudaGraph_t body = np.conditional.phGraph_out[0];
      unsigned long long c0 = t_launch_count;
      op.capturing = true;
      ok = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
           cudaSuccess;
      if (ok) {
        iteration();
        k_dev_cond<<<1, 32, 0, s>>>(G.ks.p, h, maxit);
        cudaGraph_t got;
        ok = cudaStreamEndCapture(s, &got) == cudaSuccess;
      }
      op.capturing = false;
      uncount(t_launch_count - c0);
      ok = ok && cudaGraphInstantiate(&G.loop[mode], outer, 0) == cudaSuccess;
    }
    if (outer) cudaGraphDestroy(outer);
    cudaGetLastError();
    if (!ok) {
      G.loop[mode] = nullptr;
      op.krylov_while = false;   // fall back to batched iteration graphs
      if (op.krylov_log) fprintf(stderr, "krylov: conditional WHILE graph unavailable, using batches\n");
    }
    G.loop_maxit[mode] = maxit;
  }
  if (G.x_ptr[mode] != x) throw Error(HC_ERR_ARGUMENT, "bicgstab_dev: solution buffer changed");
  int done_iters = 0;
  const int batch = op.krylov_batch;
  const bool dev_loop = op.krylov_while && G.loop[mode];
  while (true) {
    if (dev_loop) {
      HC_CUDA(cudaGraphLaunch(G.loop[mode], s));
    } else {
      for (int k = 0; k < batch; ++k) {
        HC_CUDA(cudaGraphLaunch(G.exec[mode], s));
        count_graph_launch(G.n_kernels[mode]);
      }
    }
    HC_CUDA(cudaMemcpyAsync(G.ks_host, G.ks.p, S_NSLOT * sizeof(double), cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    const double* h = G.ks_host;
    done_iters = (int)h[S_ITERS];
    if (dev_loop) count_graph_launch((G.n_kernels[mode] + 1) * (unsigned long long)std::max(done_iters, 1));
    if (h[S_ERR] != 0.0) {
      char msg[128];
      snprintf(msg, sizeof msg, "iterative linear solver stalled (breakdown %d at iteration %d)",
               (int)h[S_ERR], done_iters);
      throw Error(HC_ERR_NONCONVERGENCE, msg);
    }
    if (h[S_DONE] != 0.0) break;
    if (done_iters >= maxit) {
      char msg[160];
      snprintf(msg, sizeof msg, "iterative linear solver stalled (info=%d, relres=%.3e)", maxit,
               std::sqrt(h[S_RN2] / std::max(h[S_TOL2] / 1e-300, 1e-300)));
      throw Error(HC_ERR_NONCONVERGENCE, msg);
    }
  }
  return done_iters;
}


void krylov_append(Operator& op, GraphBuilder& gb, const double2* b, double2* x, double inv_dt, int mode,
                   const double* rtol_dev, int maxit, double* ns) {
  Work& W = work(op);
  if (!op.kg) op.kg = new KrylovGraphs();
  KrylovGraphs& G = *op.kg;
  const long long n = op.P.nvox;
  const int nb = (int)std::min<long long>((n + TPB - 1) / TPB, (long long)krylov_blocks_per_sm() * op.n_sm);
  if (!G.ks.p) {
    G.ks.alloc(S_NSLOT);
    G.part.alloc(4 * nb + 8);
    G.jpart.alloc(3 * jpart_cap(op));
    G.ticket.alloc(1);
    HC_CUDA(cudaMemset(G.ticket.p, 0, sizeof(unsigned)));
    HC_CUDA(cudaMallocHost(&G.ks_host, S_NSLOT * sizeof(double)));
  }
  cudaStream_t s = gb.s;
  double* ks = G.ks.p;
  double* part = G.part.p;
  unsigned* tk = G.ticket.p;
  // the WHILE handle is set explicitly before the node: a nested loop is re-entered in
  // every Newton iteration, while the handle default is applied once per graph launch
  cudaGraphConditionalHandle h = gb.handle(0);
  gb.capture([&] {
    HC_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double2), s));
    HC_CUDA(cudaMemcpyAsync(W.kr.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    HC_CUDA(cudaMemcpyAsync(W.khat.p, b, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    HC_CUDA(cudaMemsetAsync(W.kp.p, 0, n * sizeof(double2), s));
    HC_CUDA(cudaMemsetAsync(W.kv.p, 0, n * sizeof(double2), s));
    HC_CUDA(cudaMemsetAsync(ks, 0, S_NSLOT * sizeof(double), s));   // clears DONE of the last solve
    launch(k_dev_dot2, nb, TPB, 0, s, n, ks, b, b, nullptr, nullptr, part, -1, tk); HC_COUNT();
    launch(k_dev_init_dev, 1, 256, 0, s, nb, (const double*)part, ks, rtol_dev); HC_COUNT();
    k_dev_cond<<<1, 32, 0, s>>>(ks, h, maxit);
  });
  const SplitOut so{op.labels.p, op.P.t_plus, op.amg->rs[0].p, op.amg->rs[1].p};
  GraphBuilder body{s, gb.cond(h, cudaGraphCondTypeWhile), {}};
  body.capture([&] {
    bicgstab_iteration(op, W, G, so, x, inv_dt, mode, nb, n, s);
    k_dev_cond<<<1, 32, 0, s>>>(ks, h, maxit);
  });
  gb.capture([&] { launch(k_dev_check, 1, 1, 0, s, (const double*)ks, maxit, ns); HC_COUNT(); });
}

}  // namespace hc
