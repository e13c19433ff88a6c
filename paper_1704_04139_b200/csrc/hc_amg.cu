// Field-split, phase-aware smoothed-aggregation multigrid preconditioner.
//
// The reference factorizes the Newton Jacobian with SuperLU, or uses ILU +
// LGMRES (fvm/newton.py:75-83).  On the device the Jacobian stays matrix-free
// and the linear solve is BiCGStab preconditioned by:
//   1. the row transform T (electrolyte c row -= t+ * phi row of the same voxel),
//      which cancels the migration and chemical-potential couplings exactly;
//   2. a block lower-triangular split of T J: phi block first, then c block;
//   3. one V-cycle per block of a smoothed-aggregation multigrid whose tentative
//      aggregates are (2^l x 2^l x 2^l block, phase) pairs.  Aggregation never mixes
//      phases, so weakly coupled conductor clusters (graphite / electrolyte networks
//      joined only by Butler-Volmer faces, the metal counter stack) keep their own
//      coarse unknowns; the prolongator smoothing P = (I - w D^-1 A) P0 removes the
//      interpolation-energy defect of plain aggregation, which otherwise grows with
//      the electrode thickness.
// Sparsity patterns (A_l, P_l, P_l^T, A_l+1 = P_l^T A_l P_l) depend on the labels
// only and are built once on the host; the values are recomputed on the device for
// every linearization by deterministic per-row kernels (no atomics).  The fine level
// is applied matrix-free (jvp kernels); its CSR copy only feeds the first Galerkin
// product.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <memory>
#include <numeric>
#include <chrono>
#include <cstdio>
#include <thread>
#include <type_traits>

#include "hc_amg.cuh"
#include "hc_stencil.cuh"

namespace cg = cooperative_groups;
#include "hc_tma.cuh"

namespace hc {

namespace {
constexpr int TPB = 256;
inline int nblk(long long n, int tpb = TPB) { return (int)std::max<long long>(1, (n + tpb - 1) / tpb); }

__device__ __forceinline__ bool grounded_d(const DevParams& P, uint8_t lab, int z) {
  return z == P.nz - 1 && lab == CC;
}
__device__ __forceinline__ double harm_d(const DevParams& P, uint8_t a, uint8_t b) {
  double sa = P.sig[a], sb = P.sig[b];
  return 2.0 * sa * sb / (sa + sb) * P.gF2;
}
__device__ __forceinline__ int find_col(const int32_t* col, int lo, int hi, int32_t c) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (col[mid] < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- level 0: assemble the field block of the fine operator into CSR --------
// field 1: J_pp; field 0: (T J)_cc + mass.  One thread per voxel row.
__global__ void k_assemble0(DevParams P, int field, const uint8_t* __restrict__ lab,
                            const int32_t* __restrict__ if_rank, const int32_t* __restrict__ if_dir,
                            const int32_t* __restrict__ if_so, const int8_t* __restrict__ if_kind,
                            const double* __restrict__ coef, long long n_if, double inv_dt,
                            const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            double* __restrict__ val, double* __restrict__ dinv) {
  pdl_wait();
  int x, y, z, v;
  if (!vox_index(P, x, y, z, v)) return;
  int r0 = rp[v], r1 = rp[v + 1];
  if (r0 == r1) { dinv[v] = 0.0; return; }
  for (int k = r0; k < r1; ++k) val[k] = 0.0;
  uint8_t a = lab[v];
  const double tp = P.t_plus;
  double diag = field == 0 ? inv_dt : 0.0;
  int rk = if_rank[v];
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
    uint8_t kd = kind_of(a, b);
    bool gb = grounded_d(P, b, zb);
    double off = 0.0;
    bool has = false;
    if (field == 1) {
      if (gb) {
        if (kd == K_CONT || kd == K_CONTACT) diag += harm_d(P, a, b);
        continue;
      }
      if (kd == K_CONT) {
        double g = (a == GR ? P.sigma_gr : (a == EL ? P.kappa : P.sig[a])) * P.gF2;
        diag += g; off = -g; has = true;
      } else if (kd == K_CONTACT) {
        double g = harm_d(P, a, b);
        diag += g; off = -g; has = true;
      } else if (kd == K_BV || kd == K_CE || kd == K_STRIP) {
        double g = coef[2 * n_if + if_dir[6LL * rk + d]];
        diag += g; off = -g; has = true;
      }
    } else {
      if (gb) continue;
      if (kd == K_CONT && (a == GR || a == EL)) {
        double g = (a == GR ? P.d_gr : P.d_el) * P.inv_h2;
        diag += g; off = -g; has = true;
      } else if (kd == K_BV || kd == K_CE || kd == K_STRIP) {
        int f = if_dir[6LL * rk + d];
        double ca = coef[f], cb = coef[n_if + f];
        if (if_so[f] == (int32_t)v) {              // graphite c row
          if (if_kind[f] == IF_BV) { diag += ca; off = cb; has = true; }
        } else {                                   // electrolyte c row: -(1 - t+) dv
          diag += -(1.0 - tp) * cb;
          if (if_kind[f] == IF_BV) { off = -(1.0 - tp) * ca; has = true; }
        }
      }
    }
    if (has) val[find_col(ci, r0, r1, (int32_t)nb)] += off;
  }
  val[find_col(ci, r0, r1, (int32_t)v)] += diag;
  dinv[v] = diag != 0.0 ? 1.0 / diag : 0.0;
}

__global__ void k_dinv(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                       const double* __restrict__ v, double* __restrict__ dinv, CV* __restrict__ dinvc) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  int r0 = rp[i], r1 = rp[i + 1];
  if (r0 < r1) {
    int k = find_col(ci, r0, r1, i);
    if (k < r1 && ci[k] == i) d = v[k];
  }
  dinv[i] = d != 0.0 ? 1.0 / d : 0.0;
  if (dinvc) dinvc[i] = (CV)dinv[i];
}

// P = (I - w D^-1 A) P0 (smoothed) or P0 (tentative) — one thread per row
__global__ void k_smooth_P(int n, int smooth, double w, const int32_t* __restrict__ arp,
                           const int32_t* __restrict__ aci, const double* __restrict__ av,
                           const double* __restrict__ dinv, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ prp, const int32_t* __restrict__ pci,
                           double* __restrict__ pv) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p0 = prp[i], p1 = prp[i + 1];
  if (p0 == p1) return;
  for (int k = p0; k < p1; ++k) pv[k] = 0.0;
  const int self = find_col(pci, p0, p1, parent[i]);
  pv[self] += 1.0;
  if (!smooth) return;
  double s = -w * dinv[i];
  // filtered smoothing (smooth == 2): couplings whose aggregate is not in the row's pattern
  // (weak, cross-phase ones) are lumped onto the diagonal, A^F = A - weak + diag(weak)
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const int32_t c = parent[aci[k]];
    int q = find_col(pci, p0, p1, c);
    if (q >= p1 || pci[q] != c) q = self;
    pv[q] += s * av[k];
  }
}

// Warp-per-row variants of the two Galerkin passes.  Within one (fine row, P row) pair
// the lanes take distinct output columns (a CSR row has unique columns), so the updates
// need no atomics, and the pairs are visited in the serial kernels' order: every output
// value is summed in exactly the same order — bitwise identical, ~32x the parallelism.
__global__ void k_ap_w(int n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                       const double* __restrict__ av, const int32_t* __restrict__ prp,
                       const int32_t* __restrict__ pci, const double* __restrict__ pv,
                       const int32_t* __restrict__ qrp, const int32_t* __restrict__ qci,
                       double* __restrict__ qv) {
  pdl_wait();
  const int i = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
  const int r0 = qrp[i], r1 = qrp[i + 1];
  if (r0 == r1) return;
  for (int k = r0 + lane; k < r1; k += 32) qv[k] = 0.0;
  __syncwarp();
  for (int k = arp[i]; k < arp[i + 1]; ++k) {
    const int j = aci[k];
    const double a = av[k];
    for (int m = prp[j] + lane; m < prp[j + 1]; m += 32) qv[find_col(qci, r0, r1, pci[m])] += a * pv[m];
    __syncwarp();
  }
}

__global__ void k_ptap_w(int n_next, const int32_t* __restrict__ pt_ptr,
                         const int32_t* __restrict__ pt_row, const int32_t* __restrict__ pt_idx,
                         const double* __restrict__ pv, const int32_t* __restrict__ qrp,
                         const int32_t* __restrict__ qci, const double* __restrict__ qv,
                         const int32_t* __restrict__ nrp, const int32_t* __restrict__ nci,
                         double* __restrict__ nv) {
  pdl_wait();
  const int I = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (I >= n_next) return;
  const int r0 = nrp[I], r1 = nrp[I + 1];
  for (int k = r0 + lane; k < r1; k += 32) nv[k] = 0.0;
  __syncwarp();
  for (int q = pt_ptr[I]; q < pt_ptr[I + 1]; ++q) {
    const int i = pt_row[q];
    const double p = pv[pt_idx[q]];
    for (int m = qrp[i] + lane; m < qrp[i + 1]; m += 32) nv[find_col(nci, r0, r1, qci[m])] += p * qv[m];
    __syncwarp();
  }
}

// R = P^T A: row I is the P-weighted sum of the fine rows in P^T's row I (warp per
// coarse row, fine rows in order, the same fixed summation order as k_ptap_w)
__global__ void k_pta_w(int n_next, const int32_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_row,
                        const int32_t* __restrict__ pt_idx, const double* __restrict__ pv,
                        const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                        const double* __restrict__ av, const int32_t* __restrict__ rrp,
                        const int32_t* __restrict__ rci, double* __restrict__ rv) {
  pdl_wait();
  const int I = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (I >= n_next) return;
  const int r0 = rrp[I], r1 = rrp[I + 1];
  for (int k = r0 + lane; k < r1; k += 32) rv[k] = 0.0;
  __syncwarp();
  for (int q = pt_ptr[I]; q < pt_ptr[I + 1]; ++q) {
    const int i = pt_row[q];
    const double p = pv[pt_idx[q]];
    for (int m = arp[i] + lane; m < arp[i + 1]; m += 32) rv[find_col(rci, r0, r1, aci[m])] += p * av[m];
    __syncwarp();
  }
}

// ---- coarsest level: dense LU with partial pivoting in one CTA --------------
__global__ void k_dense_from_csr(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cl,
                                 const double* __restrict__ v, double* __restrict__ A) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < n; ++j) A[(long long)i * n + j] = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) A[(long long)i * n + cl[k]] = v[k];
}

// coarsest level: LU with partial pivoting in shared memory, then the explicit
// inverse (one thread per column), so every coarse solve is one dense mat-vec
__global__ void k_dense_inverse(int n, const double* __restrict__ A, double* __restrict__ Ainv) {
  pdl_wait();
  extern __shared__ double sm[];
  double* M = sm;                         // n x n
  int* perm = (int*)(sm + (size_t)n * n);
  __shared__ int piv_row;
  int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += blockDim.x) M[e] = A[e];
  for (int i = tid; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (tid == 0) {
      int p = k;
      double best = fabs(M[k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (fabs(M[i * n + k]) > best) { best = fabs(M[i * n + k]); p = i; }
      piv_row = p;
      if (p != k) { int t = perm[k]; perm[k] = perm[p]; perm[p] = t; }
    }
    __syncthreads();
    int p = piv_row;
    if (p != k)
      for (int j = tid; j < n; j += blockDim.x) {
        double t = M[k * n + j]; M[k * n + j] = M[p * n + j]; M[p * n + j] = t;
      }
    __syncthreads();
    double d = M[k * n + k];
    double inv = d != 0.0 ? 1.0 / d : 0.0;
    for (int i = k + 1 + tid; i < n; i += blockDim.x) M[i * n + k] *= inv;
    __syncthreads();
    int m = n - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      int i = k + 1 + e / m, j = k + 1 + e % m;
      M[i * n + j] -= M[i * n + k] * M[k * n + j];
    }
    __syncthreads();
  }
  // column j of the inverse: solve L U x = e_{perm^-1 ...}: (P A) = L U, A^-1 = U^-1 L^-1 P
  for (int j = tid; j < n; j += blockDim.x) {
    double y[HC_COARSE_MAX];
    for (int i = 0; i < n; ++i) {
      double s = perm[i] == j ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= M[i * n + k] * y[k];
      y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < n; ++k) s -= M[i * n + k] * y[k];
      double d = M[i * n + i];
      y[i] = d != 0.0 ? s / d : 0.0;
    }
    for (int i = 0; i < n; ++i) Ainv[i * n + j] = y[i];
  }
}

// x = Ainv b, one warp per row
__global__ void k_dense_matvec(int n, const double* __restrict__ Ainv, const CV* __restrict__ b,
                               CV* __restrict__ x) {
  pdl_wait();
  int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s += Ainv[row * n + j] * (double)b[j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) x[row] = (CV)s;
}

// ---- coarsest levels above HC_COARSE_MAX rows: blocked Gauss-Jordan on [A | I] in global memory.
// Pivot blocks of GJ_B rows are inverted in shared memory (k_gj_pivot_inverse); the Galerkin operators
// are diagonally dominant enough to need no pivoting;
// every block step is five launches whatever the size, so the whole inverse stays a short kernel
// chain that a graph capture can hold.
constexpr int GJ_B = 64;
__global__ void k_gj_init(int n, const double* __restrict__ A, double* __restrict__ G) {
  pdl_wait();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * 2 * n) return;
  const int i = (int)(e / (2 * n)), j = (int)(e % (2 * n));
  G[e] = j < n ? A[(long long)i * n + j] : (j - n == i ? 1.0 : 0.0);
}
// the column panel k0 .. k0 + bw of G (all rows) into C [n][bw], its diagonal block also into P [bw][bw]
__global__ void k_gj_col(int n, int k0, int bw, const double* __restrict__ G, double* __restrict__ C,
                         double* __restrict__ P) {
  pdl_wait();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * bw) return;
  const int i = (int)(e / bw), j = (int)(e % bw);
  const double v = G[(long long)i * 2 * n + k0 + j];
  C[e] = v;
  if (i >= k0 && i < k0 + bw) P[(long long)(i - k0) * bw + j] = v;
}
// inverse of one pivot block (bw <= GJ_B) in shared memory: in-place Gauss-Jordan by all 256 threads,
// two barriers per pivot (the one-CTA LU of k_dense_inverse spent ~250 us per block, most of the
// whole inverse).  No pivoting: the Galerkin operators' diagonal blocks are diagonally dominant; a
// zero pivot (a row without entries) leaves a zero row and column, like k_dense_inverse.
__global__ void __launch_bounds__(256) k_gj_pivot_inverse(int bw, const double* __restrict__ P, double* __restrict__ D) {
  pdl_wait();
  __shared__ double M[GJ_B][GJ_B + 1], colk[GJ_B], rowk[GJ_B];
  const int tid = threadIdx.x;
  for (int e = tid; e < bw * bw; e += 256) M[e / bw][e % bw] = P[e];
  for (int k = 0; k < bw; ++k) {
    __syncthreads();
    const double d = M[k][k];
    const double p = d != 0.0 ? 1.0 / d : 0.0;
    if (tid < bw) {
      colk[tid] = M[tid][k];
      rowk[tid] = (tid == k ? 1.0 : M[k][tid]) * p;
    }
    __syncthreads();
    for (int e = tid; e < bw * bw; e += 256) {
      const int i = e / bw, j = e - i * bw;
      M[i][j] = i == k ? rowk[j] : (j == k ? 0.0 : M[i][j]) - colk[i] * rowk[j];
    }
  }
  __syncthreads();
  for (int e = tid; e < bw * bw; e += 256) D[e] = M[e / bw][e % bw];
}
// Out[i][j] = beta Out[i][j] + alpha sum_k A[i][k] B[k][j] for rows i < m outside [skip0, skip0 + skipn),
// columns j0 <= j < j1 (A [m][kd], B and Out with leading dimension ld): 128 x 64 tiles, 8 x 4 per
// thread, operands staged per 16-deep k chunk and read back as double2 (the 16 threads of a row
// group share their A values: broadcast loads)
constexpr int GJ_TM = 128, GJ_TN = 64, GJ_KC = 16;
__global__ void __launch_bounds__(256) k_gj_gemm(int m, int kd, int j0, int j1, int ld, double alpha,
                                                const double* __restrict__ A, const double* __restrict__ B,
                                                double beta, double* __restrict__ Out, int skip0, int skipn) {
  pdl_wait();
  __shared__ __align__(16) double As[GJ_KC][GJ_TM + 2], Bs[GJ_KC][GJ_TN];
  const int i0 = blockIdx.y * GJ_TM, c0 = j0 + blockIdx.x * GJ_TN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[8][4] = {};
  for (int kc = 0; kc < kd; kc += GJ_KC) {
    const int kn = min(GJ_KC, kd - kc);
    for (int e = threadIdx.x; e < GJ_TM * GJ_KC; e += 256) {   // A tile: k fastest in memory
      const int r = e / GJ_KC, k = e % GJ_KC;
      As[k][r] = (k < kn && i0 + r < m) ? A[(long long)(i0 + r) * kd + kc + k] : 0.0;
    }
    for (int e = threadIdx.x; e < GJ_KC * GJ_TN; e += 256) {
      const int k = e / GJ_TN, c = e % GJ_TN;
      Bs[k][c] = (k < kn && c0 + c < j1) ? B[(long long)(kc + k) * ld + c0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < GJ_KC; ++k) {
      double a[8], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 t = *reinterpret_cast<const double2*>(&As[k][ty * 8 + 2 * q]);
        a[2 * q] = t.x;
        a[2 * q + 1] = t.y;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 t = *reinterpret_cast<const double2*>(&Bs[k][tx * 4 + 2 * q]);
        b[2 * q] = t.x;
        b[2 * q + 1] = t.y;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[q][r] = fma(a[q], b[r], acc[q][r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + ty * 8 + q;
    if (i >= m || (i >= skip0 && i < skip0 + skipn)) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int j = c0 + tx * 4 + r;
      if (j < j1) {
        double* o = Out + (long long)i * ld + j;
        *o = (beta != 0.0 ? beta * *o : 0.0) + alpha * acc[q][r];
      }
    }
  }
}
// rows k0 .. k0 + bw of G, columns j0 .. j1, from R (same leading dimension)
__global__ void k_gj_row(int n, int k0, int bw, int j0, int j1, const double* __restrict__ R, double* __restrict__ G) {
  pdl_wait();
  const int w = j1 - j0;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)bw * w) return;
  const int i = (int)(e / w), j = j0 + (int)(e % w);
  G[(long long)(k0 + i) * 2 * n + j] = R[(long long)i * 2 * n + j];
}
__global__ void k_gj_out(int n, const double* __restrict__ G, double* __restrict__ Ainv) {
  pdl_wait();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e / n), j = (int)(e % n);
  Ainv[e] = G[(long long)i * 2 * n + n + j];
}

// ---- cycle kernels ------------------------------------------------------------

__global__ void k_csr_smooth0(int n, double w, const CV* __restrict__ dinv,
                              const CV* __restrict__ b, CV* __restrict__ x) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = w * dinv[i] * b[i];
}

__global__ void k_to_float(long long n, const double* __restrict__ a, float* __restrict__ b) {
  pdl_wait();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

// sliced-ELL values from the CSR fp32 values (after every numeric setup)
__global__ void k_sell_gather(long long n, const int32_t* __restrict__ map, const float* __restrict__ vf,
                              float* __restrict__ out) {
  pdl_wait();
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q < n) {
    const int m = map[q];
    out[q] = m >= 0 ? vf[m] : 0.0f;
  }
}

// The k_csr_x sweep on the sliced-ELL copy: T lanes per row, a warp per slice of 32 / T
// rows; entry j of slice row r sits at base + ((j / T) * (32 / T) + r) * T + j % T, so every
// k-step of the warp is one coalesced 32-entry load and the rows' k-th columns (mostly
// consecutive) are gathered together; the T partial sums are combined by shuffles
template <int T, int XM>
__global__ void k_sell_x(int n, double w, double alpha, const int32_t* __restrict__ sp,
                         const int32_t* __restrict__ sc, const float* __restrict__ sv,
                         const CV* __restrict__ dinv, const CV* __restrict__ b,
                         const CV* __restrict__ x, const int32_t* __restrict__ parent,
                         const CV* __restrict__ xc, CV* __restrict__ y, int resid,
                         CV* __restrict__ x0) {
  pdl_wait();
  constexpr int R = 32 / T;   // rows per slice
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int slice = (int)(gt >> 5);
  if ((long long)slice * R >= n) return;
  const int lane = threadIdx.x & 31;
  const int i = slice * R + lane / T;
  auto xin = [&](int j) -> double {
    if (XM == 0) return (double)x[j];
    if (XM == 1) return w * (double)dinv[j] * (double)b[j];
    return (double)x[j] + alpha * (double)xc[parent[j]];
  };
  const int base = sp[slice], width = (sp[slice + 1] - base) >> 5;   // k-steps of 32 entries
  const int32_t* cp = sc + base + lane;
  const float* vp = sv + base + lane;
  double s = 0.0;
  int k = 0;
  for (; k + 3 < width; k += 4) {
    const int c0 = cp[0], c1 = cp[32], c2 = cp[64], c3 = cp[96];
    const double a0 = vp[0], a1 = vp[32], a2 = vp[64], a3 = vp[96];
    const double x0_ = xin(c0), x1 = xin(c1), x2 = xin(c2), x3 = xin(c3);
    s += a0 * x0_;
    s += a1 * x1;
    s += a2 * x2;
    s += a3 * x3;
    cp += 128;
    vp += 128;
  }
  for (; k < width; ++k, cp += 32, vp += 32) s += (double)*vp * xin(*cp);
#pragma unroll
  for (int o = T / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, T);
  if (lane % T == 0 && i < n) {
    const double xi = xin(i), bi = b[i];
    y[i] = (CV)(resid ? bi - s : xi + w * (double)dinv[i] * (bi - s));
    if (x0) x0[i] = (CV)xi;
  }
}

// packed entries of a level operator from its fp64 values (after every numeric setup):
// off-diagonals rounded to bf16 (nearest even), the diagonal entry's value 0, the row's
// rounding errors folded into the fp32 diagonal kept per row
__global__ void k_pack_rows(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ a, const uint16_t* __restrict__ off,
                            uint32_t* __restrict__ pk, float* __restrict__ diag) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double err = 0.0, d = 0.0;
  for (int q = rp[i]; q < rp[i + 1]; ++q) {
    const double aq = a[q];
    if (ci[q] == i) {
      d += aq;
      pk[q] = off[q];
      continue;
    }
    unsigned u = __float_as_uint((float)aq);
    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
    err += aq - (double)__uint_as_float(u);
    pk[q] = u | off[q];
  }
  diag[i] = (float)(d + err);
}
// the same into the sparsified pattern (AmgLevel::As): kept entries packed in order, every
// other entry of the row lumped onto the diagonal
__global__ void k_pack_rows_sp(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               const double* __restrict__ a, const uint8_t* __restrict__ keep,
                               const int32_t* __restrict__ rps, const uint16_t* __restrict__ offs,
                               uint32_t* __restrict__ pks, float* __restrict__ diag) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double err = 0.0, d = 0.0;
  int qs = rps[i];
  for (int q = rp[i]; q < rp[i + 1]; ++q) {
    const double aq = a[q];
    if (!keep[q]) {
      err += aq;
      continue;
    }
    if (ci[q] == i) {
      d += aq;
      pks[qs] = offs[qs];
    } else {
      unsigned u = __float_as_uint((float)aq);
      u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
      err += aq - (double)__uint_as_float(u);
      pks[qs] = u | offs[qs];
    }
    ++qs;
  }
  diag[i] = (float)(d + err);
}
// sliced-ELL packed entries from the CSR packed entries
__global__ void k_sell_pack(long long n, const int32_t* __restrict__ map, const uint16_t* __restrict__ off,
                            const uint32_t* __restrict__ pk, uint32_t* __restrict__ out) {
  pdl_wait();
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q < n) {
    const int m = map[q];
    out[q] = (m >= 0 ? (pk[m] & 0xffff0000u) : 0u) | off[q];
  }
}

// k_sell_x on the packed copy: one 32-bit load per entry (bf16 value | column offset from
// the slice's base column); the diagonal comes from the per-row fp32 array
template <int T, int XM>
__global__ void k_sell_xp(int n, double w, double alpha, const int32_t* __restrict__ sp,
                          const int32_t* __restrict__ sbase, const uint32_t* __restrict__ se,
                          const float* __restrict__ diag, const CV* __restrict__ dinv,
                          const CV* __restrict__ b, const CV* __restrict__ x,
                          const int32_t* __restrict__ parent, const CV* __restrict__ xc,
                          CV* __restrict__ y, int resid, CV* __restrict__ x0) {
  pdl_wait();
  constexpr int R = 32 / T;   // rows per slice
  const long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int slice = (int)(gt >> 5);
  if ((long long)slice * R >= n) return;
  const int lane = threadIdx.x & 31;
  const int i = slice * R + lane / T;
  auto xin = [&](int j) -> double {
    if (XM == 0) return (double)x[j];
    if (XM == 1) return w * (double)dinv[j] * (double)b[j];
    return (double)x[j] + alpha * (double)xc[parent[j]];
  };
  const int base = sp[slice], width = (sp[slice + 1] - base) >> 5;   // k-steps of 32 entries
  const int cb = sbase[slice];
  const uint32_t* ep = se + base + lane;
  double s = 0.0;
  int k = 0;
  for (; k + 3 < width; k += 4) {
    const uint32_t e0 = ep[0], e1 = ep[32], e2 = ep[64], e3 = ep[96];
    const double x0_ = xin(cb + (int)(e0 & 0xffffu)), x1 = xin(cb + (int)(e1 & 0xffffu));
    const double x2 = xin(cb + (int)(e2 & 0xffffu)), x3 = xin(cb + (int)(e3 & 0xffffu));
    s += (double)__uint_as_float(e0 & 0xffff0000u) * x0_;
    s += (double)__uint_as_float(e1 & 0xffff0000u) * x1;
    s += (double)__uint_as_float(e2 & 0xffff0000u) * x2;
    s += (double)__uint_as_float(e3 & 0xffff0000u) * x3;
    ep += 128;
  }
  for (; k < width; ++k, ep += 32) {
    const uint32_t e = *ep;
    s += (double)__uint_as_float(e & 0xffff0000u) * xin(cb + (int)(e & 0xffffu));
  }
#pragma unroll
  for (int o = T / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, T);
  if (lane % T == 0 && i < n) {
    const double xi = xin(i), bi = b[i];
    s += (double)diag[i] * xi;
    y[i] = (CV)(resid ? bi - s : xi + w * (double)dinv[i] * (bi - s));
    if (x0) x0[i] = (CV)xi;
  }
}

// k_csr_x on the packed copy (column offsets from the row's smallest column)
template <int VS, int XM>
__global__ void k_csr_xp(int n, double w, double alpha, const int32_t* __restrict__ rp,
                         const int32_t* __restrict__ rbase, const uint32_t* __restrict__ pe,
                         const float* __restrict__ diag, const CV* __restrict__ dinv,
                         const CV* __restrict__ b, const CV* __restrict__ x,
                         const int32_t* __restrict__ parent, const CV* __restrict__ xc,
                         CV* __restrict__ y, int resid, CV* __restrict__ x0) {
  pdl_wait();
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int i = (int)(gt / VS), lane = (int)(gt % VS);
  if (i >= n) return;
  auto xin = [&](int j) -> double {
    if (XM == 0) return (double)x[j];
    if (XM == 1) return w * (double)dinv[j] * (double)b[j];
    return (double)x[j] + alpha * (double)xc[parent[j]];
  };
  double s = 0.0;
  const int k1 = rp[i + 1], cb = rbase[i];
  int k = rp[i] + lane;
  for (; k + 3 * VS < k1; k += 4 * VS) {
    const uint32_t e0 = pe[k], e1 = pe[k + VS], e2 = pe[k + 2 * VS], e3 = pe[k + 3 * VS];
    const double x0_ = xin(cb + (int)(e0 & 0xffffu)), x1 = xin(cb + (int)(e1 & 0xffffu));
    const double x2 = xin(cb + (int)(e2 & 0xffffu)), x3 = xin(cb + (int)(e3 & 0xffffu));
    s += (double)__uint_as_float(e0 & 0xffff0000u) * x0_;
    s += (double)__uint_as_float(e1 & 0xffff0000u) * x1;
    s += (double)__uint_as_float(e2 & 0xffff0000u) * x2;
    s += (double)__uint_as_float(e3 & 0xffff0000u) * x3;
  }
  for (; k < k1; k += VS) {
    const uint32_t e = pe[k];
    s += (double)__uint_as_float(e & 0xffff0000u) * xin(cb + (int)(e & 0xffffu));
  }
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, VS);
  if (lane == 0) {
    const double xi = xin(i), bi = b[i];
    s += (double)diag[i] * xi;
    y[i] = (CV)(resid ? bi - s : xi + w * (double)dinv[i] * (bi - s));
    if (x0) x0[i] = (CV)xi;
  }
}

// VS lanes per row (VS = 1, 8 or 32), chosen per level from the mean row length
template <int VS, class VT>
__global__ void k_csr_jacobi_v(int n, double w, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ cl, const VT* __restrict__ v,
                               const CV* __restrict__ dinv, const CV* __restrict__ b,
                               const CV* __restrict__ x, CV* __restrict__ y, int resid) {
  pdl_wait();
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int i = (int)(gt / VS), lane = (int)(gt % VS);
  if (i >= n) return;
  double s = 0.0;
  const int k1 = rp[i + 1];
  int k = rp[i] + lane;
  double s2 = 0.0;
  for (; k + VS < k1; k += 2 * VS) {   // two independent gathers in flight per lane
    const int c0 = cl[k], c1 = cl[k + VS];
    const double a0 = (double)v[k], a1 = (double)v[k + VS];
    s += a0 * (double)x[c0];
    s2 += a1 * (double)x[c1];
  }
  if (k < k1) s += (double)v[k] * (double)x[cl[k]];
  s += s2;
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, VS);
  if (lane == 0) y[i] = (CV)(resid ? (double)b[i] - s : (double)x[i] + w * (double)dinv[i] * ((double)b[i] - s));
}

// Generalized sweep: y = xin + w D^-1 (b - A xin)  (resid: y = b - A xin) where the
// input vector is materialised on the fly:
//   XM 0: xin = x                                  (plain sweep)
//   XM 1: xin = w D^-1 b                           (first pre-sweep from a zero guess)
//   XM 2: xin = x + alpha * xc[parent]             (first post-sweep fused with the
//                                                   tentative-prolongator correction)
template <int VS, class VT, int XM>
__global__ void k_csr_x(int n, double w, double alpha, const int32_t* __restrict__ rp,
                        const int32_t* __restrict__ cl, const VT* __restrict__ v,
                        const CV* __restrict__ dinv, const CV* __restrict__ b,
                        const CV* __restrict__ x, const int32_t* __restrict__ parent,
                        const CV* __restrict__ xc, CV* __restrict__ y, int resid,
                        CV* __restrict__ x0) {
  pdl_wait();
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int i = (int)(gt / VS), lane = (int)(gt % VS);
  if (i >= n) return;
  auto xin = [&](int j) -> double {
    if (XM == 0) return (double)x[j];
    if (XM == 1) return w * (double)dinv[j] * (double)b[j];
    return (double)x[j] + alpha * (double)xc[parent[j]];
  };
  double s = 0.0;
  // four nonzeros per trip with all index / value loads issued before the gathers (the
  // rows are short, so a one-at-a-time loop is a chain of dependent L2 round trips);
  // the summation order is the plain loop's
  const int k1 = rp[i + 1];
  int k = rp[i] + lane;
  for (; k + 3 * VS < k1; k += 4 * VS) {
    const int c0 = cl[k], c1 = cl[k + VS], c2 = cl[k + 2 * VS], c3 = cl[k + 3 * VS];
    const double a0 = (double)v[k], a1 = (double)v[k + VS], a2 = (double)v[k + 2 * VS], a3 = (double)v[k + 3 * VS];
    const double x0 = xin(c0), x1 = xin(c1), x2 = xin(c2), x3 = xin(c3);
    s += a0 * x0;
    s += a1 * x1;
    s += a2 * x2;
    s += a3 * x3;
  }
  for (; k < k1; k += VS) s += (double)v[k] * xin(cl[k]);
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, VS);
  if (lane == 0) {
    const double xi = xin(i), bi = b[i];
    y[i] = (CV)(resid ? bi - s : xi + w * (double)dinv[i] * (bi - s));
    if (x0) x0[i] = (CV)xi;   // residual of the zero-guess iterate: also store that iterate
  }
}

template <class TV>
__global__ void k_csr_prolong(int n, double alpha, const int32_t* __restrict__ prp,
                              const int32_t* __restrict__ pci, const TV* __restrict__ pv,
                              const CV* __restrict__ xn, CV* __restrict__ x) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int m = prp[i]; m < prp[i + 1]; ++m) s += (double)pv[m] * (double)xn[pci[m]];
  x[i] = (CV)((double)x[i] + alpha * s);
}

__global__ void k_vec_add(int n, const CV* __restrict__ a, CV* __restrict__ x) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (CV)((double)x[i] + (double)a[i]);
}

// b[I] = sum_q ptv[q] res[pt_row[q]] (P^T res), 8 lanes per coarse row; res is the fine
// level's fp64 residual (RT double) or a coarse level's (RT = CV)
template <class TV, class RT>
__global__ void k_restrict_v(int n1, const int32_t* __restrict__ pt_ptr,
                             const int32_t* __restrict__ pt_row, const TV* __restrict__ ptv,
                             const RT* __restrict__ res, CV* __restrict__ b1) {
  pdl_wait();
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int I = (int)(gt >> 3), lane = (int)(gt & 7);
  if (I >= n1) return;
  double s = 0.0;
  const int q1 = pt_ptr[I + 1];
  int q = pt_ptr[I] + lane;
  for (; q + 8 < q1; q += 16) {
    const int r0 = pt_row[q], r1 = pt_row[q + 8];
    const double a0 = (double)ptv[q], a1 = (double)ptv[q + 8];
    const double x0 = res[r0], x1 = res[r1];
    s += a0 * x0;
    s += a1 * x1;
  }
  for (; q < q1; q += 8) s += (double)ptv[q] * (double)res[pt_row[q]];
  s += __shfl_down_sync(0xffffffffu, s, 4, 8);
  s += __shfl_down_sync(0xffffffffu, s, 2, 8);
  s += __shfl_down_sync(0xffffffffu, s, 1, 8);
  if (lane == 0) b1[I] = (CV)s;
}
// fused residual + restriction for a tentative prolongator: b1[I] = sum of b over the
// aggregate's members - (R x)_I with R = P^T A (VS lanes per coarse row)
template <int VS, class VT>
__global__ void k_resid_restrict(int n1, const int32_t* __restrict__ pt_ptr, const int32_t* __restrict__ pt_row,
                                 const int32_t* __restrict__ rrp, const int32_t* __restrict__ rci,
                                 const VT* __restrict__ rv, const VT* __restrict__ ptv,
                                 const CV* __restrict__ b, const CV* __restrict__ x,
                                 CV* __restrict__ b1) {
  pdl_wait();
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int I = (int)(gt / VS), lane = (int)(gt % VS);
  const bool ok = I < n1;
  double s = 0.0;
  if (ok) {
    const int k1 = rrp[I + 1];
    int k = rrp[I] + lane;
    for (; k + 3 * VS < k1; k += 4 * VS) {
      const int c0 = rci[k], c1 = rci[k + VS], c2 = rci[k + 2 * VS], c3 = rci[k + 3 * VS];
      const double a0 = (double)rv[k], a1 = (double)rv[k + VS], a2 = (double)rv[k + 2 * VS], a3 = (double)rv[k + 3 * VS];
      const double x0 = x[c0], x1 = x[c1], x2 = x[c2], x3 = x[c3];
      s -= a0 * x0;
      s -= a1 * x1;
      s -= a2 * x2;
      s -= a3 * x3;
    }
    for (; k < k1; k += VS) s -= (double)rv[k] * (double)x[rci[k]];
    for (int q = pt_ptr[I] + lane; q < pt_ptr[I + 1]; q += VS) s += (double)ptv[q] * (double)b[pt_row[q]];
  }
#pragma unroll
  for (int o = VS / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, VS);
  if (ok && lane == 0) b1[I] = (CV)s;
}

__global__ void k_gather_ptv(long long n, const int32_t* __restrict__ pt_idx,
                             const double* __restrict__ pv, double* __restrict__ ptv) {
  pdl_wait();
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q < n) ptv[q] = pv[pt_idx[q]];
}
template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(h.size());
  if (!h.empty()) HC_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// host CSR pattern
struct HPat {
  std::vector<int32_t> rp, ci;
  int n() const { return (int)rp.size() - 1; }
};

template <class F>
void parallel_for(int n, F&& f) {
  int nt = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 4096) nt = 1;
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      int lo = (int)((long long)n * t / nt), hi = (int)((long long)n * (t + 1) / nt);
      for (int i = lo; i < hi; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

// rows given as per-row vectors -> CSR (sorted, unique)
HPat finish(std::vector<std::vector<int32_t>>& rows) {
  HPat p;
  p.rp.assign(rows.size() + 1, 0);
  parallel_for((int)rows.size(), [&](int i) {
    auto& r = rows[i];
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
  });
  for (size_t i = 0; i < rows.size(); ++i) p.rp[i + 1] = p.rp[i] + (int32_t)rows[i].size();
  p.ci.resize(p.rp.back());
  parallel_for((int)rows.size(), [&](int i) {
    std::copy(rows[i].begin(), rows[i].end(), p.ci.begin() + p.rp[i]);
  });
  return p;
}

void upload_csr(Csr& c, const HPat& p) {
  c.n = p.n();
  c.nnz = (long long)p.ci.size();
  upload(c.rp, p.rp);
  upload(c.ci, p.ci);
  c.v.alloc(std::max<size_t>(p.ci.size(), 1));
  c.vf.alloc(std::max<size_t>(p.ci.size(), 1));
}

}  // namespace

// packed-entry patterns of a level operator (see Csr::pk_*): per-row / per-slice base column
// and 16-bit offsets; leaves pk_ok false when some row or slice spans 65536 columns or more
static void build_packed(Csr& c, const HPat& p) {
  const int n = p.n();
  c.pk_ok = false;
  if (!n || p.ci.empty()) return;
  std::vector<int32_t> base(n);
  std::vector<uint16_t> off(p.ci.size());
  for (int i = 0; i < n; ++i) {
    int lo = i, hi = i;
    for (int q = p.rp[i]; q < p.rp[i + 1]; ++q) {
      lo = std::min(lo, p.ci[q]);
      hi = std::max(hi, p.ci[q]);
    }
    if (hi - lo >= 65536) return;
    base[i] = lo;
    for (int q = p.rp[i]; q < p.rp[i + 1]; ++q) off[q] = (uint16_t)(p.ci[q] - lo);
  }
  upload(c.pk_base, base);
  upload(c.pk_off, off);
  c.pk.alloc(p.ci.size());
  c.pk_diag.alloc(n);
  c.pk_ok = true;
}
// the same for the sliced-ELL copy (after build_sell): offsets from the slice's smallest column
static void build_packed_sell(Csr& c, const std::vector<int32_t>& ptr, const std::vector<int32_t>& col) {
  if (!c.pk_ok) return;
  const int ns = (int)ptr.size() - 1;
  std::vector<int32_t> base(ns);
  std::vector<uint16_t> off(col.size());
  for (int sl = 0; sl < ns; ++sl) {
    int lo = INT32_MAX, hi = 0;
    for (int q = ptr[sl]; q < ptr[sl + 1]; ++q) {
      lo = std::min(lo, col[q]);
      hi = std::max(hi, col[q]);
    }
    if (ptr[sl + 1] > ptr[sl] && hi - lo >= 65536) {
      c.sl_base.n = 0;
      return;
    }
    base[sl] = ptr[sl + 1] > ptr[sl] ? lo : 0;
    for (int q = ptr[sl]; q < ptr[sl + 1]; ++q) off[q] = (uint16_t)(col[q] - base[sl]);
  }
  upload(c.sl_base, base);
  upload(c.sl_off, off);
  c.sl_pk.alloc(std::max<size_t>(col.size(), 1));
}

// sliced-ELL pattern (see Csr::sl_*, k_sell_x) with T lanes per row from a host CSR pattern
static void build_sell(Csr& c, const HPat& p, int T) {
  const int R = 32 / T;
  const int n = p.n(), ns = (n + R - 1) / R;
  std::vector<int32_t> ptr(ns + 1, 0);
  for (int sl = 0; sl < ns; ++sl) {
    int wmax = 0;
    for (int r = sl * R; r < std::min(n, sl * R + R); ++r) wmax = std::max(wmax, p.rp[r + 1] - p.rp[r]);
    ptr[sl + 1] = ptr[sl] + 32 * ((wmax + T - 1) / T);
  }
  std::vector<int32_t> col(ptr[ns]), map(ptr[ns]);
  for (int sl = 0; sl < ns; ++sl) {
    const int width = (ptr[sl + 1] - ptr[sl]) / 32;
    for (int r = 0; r < R; ++r) {
      const int i = sl * R + r;
      const int len = i < n ? p.rp[i + 1] - p.rp[i] : 0;
      for (int k = 0; k < width; ++k)
        for (int t = 0; t < T; ++t) {
          const int j = k * T + t;
          const int q = ptr[sl] + (k * R + r) * T + t;
          if (j < len) {
            col[q] = p.ci[p.rp[i] + j];
            map[q] = p.rp[i] + j;
          } else {
            col[q] = i < n ? i : n - 1;   // (rows past the end: any valid column near the slice's)
            map[q] = -1;
          }
        }
    }
  }
  c.sl_t = T;
  upload(c.sl_ptr, ptr);
  upload(c.sl_col, col);
  upload(c.sl_map, map);
  c.sl_vf.alloc(std::max<size_t>(col.size(), 1));
  c.sl_nnz = (long long)col.size();
  c.sl_n = n;
  build_packed_sell(c, ptr, col);
}

// ============================================================== host: patterns
static void build_block(const Operator& op, const std::vector<uint8_t>& lab, int field,
                        const Amg& cfg, AmgBlock& B) {
  const int nx = op.P.nx, ny = op.P.ny, nz = op.P.nz;
  const long long nxy = (long long)nx * ny, nvox = nxy * nz;
  B.field = field;
  B.alpha = cfg.alpha;
  B.levels.clear();
  // rows of the dense coarsest level: cfg.coarse_max if set, else by grid size — its inverse costs
  // O(n^3) per hierarchy refresh, which small cells amortise over cheap steps (measured: batched
  // 48 x 48 x 96 cells 269 cell-steps/s at 1600 rows against 253 at 4000; medium and large cells
  // 13.7 / 59.7 ms per step at 4000 against 14.0 / 61.3 at 1600 / 1200)
  const int coarse_rows = cfg.coarse_max > 0
                              ? cfg.coarse_max
                              : (int)std::min<long long>(4000, std::max<long long>(1600, nvox / 128));
  auto in_field = [&](long long v) {
    uint8_t a = lab[v];
    if (field == 0) return a == GR || a == EL;
    return !((v / nxy) == nz - 1 && a == CC);
  };
  // ---- level 0 pattern from the fine couplings (same rules as k_assemble0)
  HPat A, G;
  {
    std::vector<std::vector<int32_t>> rows(nvox), grows(nvox);
    parallel_for((int)nvox, [&](int vi) {
      long long v = vi;
      if (!in_field(v)) return;
      auto& r = rows[v];
      r.push_back((int32_t)v);
      long long x = v % nx, y = (v / nx) % ny, z = v / nxy;
      uint8_t a = lab[v];
      for (int d = 0; d < 6; ++d) {
        long long nb;
        if (d == 0) { if (x == 0) continue; nb = v - 1; }
        else if (d == 1) { if (x + 1 >= nx) continue; nb = v + 1; }
        else if (d == 2) { if (y == 0) continue; nb = v - nx; }
        else if (d == 3) { if (y + 1 >= ny) continue; nb = v + nx; }
        else if (d == 4) { if (z == 0) continue; nb = v - nxy; }
        else { if (z + 1 >= nz) continue; nb = v + nxy; }
        if (!in_field(nb)) continue;
        uint8_t kd = kind_of(a, lab[nb]);
        if (kd == K_CONT) grows[v].push_back((int32_t)nb);   // same-phase conduction: strong
        bool has = field == 1 ? (kd == K_CONT || kd == K_CONTACT || kd == K_BV || kd == K_CE ||
                                 kd == K_STRIP)
                              : ((kd == K_CONT) || kd == K_BV);
        if (has) r.push_back((int32_t)nb);
      }
    });
    A = finish(rows);
    G = finish(grows);
  }
  // per-row geometry for aggregation: block coordinates and phase (-1 = empty row)
  std::vector<int32_t> bx(nvox), by(nvox), bz(nvox), ph(nvox);
  for (long long v = 0; v < nvox; ++v) {
    bx[v] = (int32_t)(v % nx);
    by[v] = (int32_t)((v / nx) % ny);
    bz[v] = (int32_t)(v / nxy);
    ph[v] = in_field(v) ? lab[v] : -1;
  }
  int sx = nx, sy = ny, sz = nz;
  int level = 0;
  while (true) {
    B.levels.emplace_back();
    AmgLevel& L = B.levels.back();
    const int n = A.n();
    L.n = n;
    upload_csr(L.A, A);
    if (level >= 1 && cfg.pack && n > 0) build_packed(L.A, A);
    if (level >= 1 && cfg.sell_max_avg > 0 && n > 0) {
      // lanes per row: enough that each lane keeps ~sell_lane_nnz entries, and enough
      // threads in flight (n T >= sell_min_rows) for the sliced copy to pay
      const double avg = (double)A.ci.size() / n;
      int T = 1;
      while (T < 32 && avg / T > cfg.sell_lane_nnz) T *= 2;
      if (cfg.sell_force_t) T = cfg.sell_force_t;
      if ((long long)n * T >= cfg.sell_min_rows && avg <= cfg.sell_max_avg) build_sell(L.A, A, T);
    }
    L.dinv.alloc(std::max(n, 1));
    int active = 0;
    for (int i = 0; i < n; ++i) active += A.rp[i + 1] > A.rp[i];
    bool can = sx > 1 || sy > 1 || sz > 1;
    // stop at the first aggregated level small enough for the dense inverse (the voxel-indexed fine
    // level only when it is tiny: a one-level hierarchy is a plain Jacobi sweep)
    const int stop = level >= 1 ? coarse_rows : std::min(coarse_rows, 128);
    if ((active <= stop && n <= HC_COARSE_CAP) || !can) break;
    // tentative aggregation: connected components (in the strong same-phase graph G)
    // of the unknowns sharing a (2x2x2 block, phase) key
    const int cf = level == 0 ? 2 : cfg.coarsen;   // block growth factor of this transfer
    int nx2 = (sx + cf - 1) / cf, ny2 = (sy + cf - 1) / cf, nz2 = (sz + cf - 1) / cf;
    std::vector<long long> key(n, -1);
    for (int i = 0; i < n; ++i)
      if (ph[i] >= 0)
        key[i] = (((long long)(bz[i] / cf) * ny2 + by[i] / cf) * nx2 + bx[i] / cf) * N_PHASES + ph[i];
    std::vector<int32_t> uf(n);
    std::iota(uf.begin(), uf.end(), 0);
    // connectivity splitting keeps disconnected same-phase pieces apart; at the top of
    // the hierarchy (few blocks left) pieces are merged so the coarsest level stays small
    const bool split = (long long)nx2 * ny2 * nz2 > 64;
    auto find = [&](int32_t i) {
      while (uf[i] != i) { uf[i] = uf[uf[i]]; i = uf[i]; }
      return i;
    };
    for (int i = 0; i < n; ++i) {
      if (key[i] < 0) continue;
      for (int k = G.rp[i]; k < G.rp[i + 1]; ++k) {
        int j = G.ci[k];
        if (key[j] != key[i]) continue;
        int a_ = find(i), b_ = find(j);
        if (!split) continue;
        if (a_ != b_) uf[std::max(a_, b_)] = std::min(a_, b_);
      }
    }
    std::vector<std::pair<long long, int32_t>> order;
    order.reserve(n);
    for (int i = 0; i < n; ++i)
      if (key[i] >= 0) order.emplace_back(key[i], split ? find(i) : 0);
    std::vector<int32_t> parent(n, -1);
    int nn = 0;
    std::vector<int32_t> nbx, nby, nbz, nph;
    {
      std::vector<std::pair<std::pair<long long, int32_t>, int32_t>> tup;
      tup.reserve(order.size());
      for (int i = 0, q = 0; i < n; ++i)
        if (key[i] >= 0) tup.push_back({order[q++], i});
      std::sort(tup.begin(), tup.end());
      for (size_t q = 0; q < tup.size(); ++q) {
        if (q == 0 || tup[q].first != tup[q - 1].first) {
          long long k = tup[q].first.first;
          long long blk = k / N_PHASES;
          nph.push_back((int32_t)(k % N_PHASES));
          nbx.push_back((int32_t)(blk % nx2));
          nby.push_back((int32_t)((blk / nx2) % ny2));
          nbz.push_back((int32_t)(blk / ((long long)nx2 * ny2)));
          ++nn;
        }
        parent[tup[q].second] = nn - 1;
      }
    }
    // strong graph of the next level: quotient of G by the aggregation
    HPat Gn;
    {
      std::vector<std::vector<int32_t>> rows(nn);
      for (int i = 0; i < n; ++i) {
        if (parent[i] < 0) continue;
        for (int k = G.rp[i]; k < G.rp[i + 1]; ++k) {
          int pj = parent[G.ci[k]];
          if (pj >= 0 && pj != parent[i]) rows[parent[i]].push_back(pj);
        }
      }
      Gn = finish(rows);
    }
    upload(L.parent, parent);
    // prolongator pattern: parent(i) plus (smoothed) the parents of row i's columns
    const int sa_c = cfg.sa_levels_c >= 0 ? cfg.sa_levels_c : (nvox <= 2000000LL ? 1 : 0);
    const bool smooth = level < (field == 0 ? sa_c : cfg.sa_levels) ||
                        (field != 0 && (cfg.sa_any ? level >= cfg.sa_levels : level == cfg.sa_levels) &&
                         n >= cfg.sa_rows_min && n <= cfg.sa_rows);
    // filtered smoothing: the prolongator reaches only the aggregates of strong (same-phase
    // connectivity graph G) neighbours
    const bool filt = smooth && field != 0 && level < 30 && ((cfg.sa_filter >> level) & 1);
    L.smoothed = smooth;
    L.filtered = filt;
    HPat Pp;
    {
      std::vector<std::vector<int32_t>> rows(n);
      parallel_for(n, [&](int i) {
        if (parent[i] < 0) return;
        rows[i].push_back(parent[i]);
        if (smooth)
          for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int j = A.ci[k];
            if (filt && j != i && !std::binary_search(G.ci.begin() + G.rp[i], G.ci.begin() + G.rp[i + 1], j))
              continue;
            if (parent[j] >= 0) rows[i].push_back(parent[j]);
          }
      });
      Pp = finish(rows);
    }
    upload_csr(L.P, Pp);
    // transpose lists of P
    std::vector<int32_t> tp(nn + 1, 0), trow(Pp.ci.size()), tidx(Pp.ci.size());
    for (int32_t c : Pp.ci) tp[c + 1]++;
    for (int I = 0; I < nn; ++I) tp[I + 1] += tp[I];
    {
      std::vector<int32_t> fill(tp.begin(), tp.end() - 1);
      for (int i = 0; i < n; ++i)
        for (int m = Pp.rp[i]; m < Pp.rp[i + 1]; ++m) {
          int q = fill[Pp.ci[m]]++;
          trow[q] = i;
          tidx[q] = m;
        }
    }
    upload(L.pt_ptr, tp);
    upload(L.pt_row, trow);
    upload(L.pt_idx, tidx);
    if (level >= 1 && cfg.fuse_restrict && (!smooth || cfg.fuse_restrict_sa)) {
      // R = P^T A pattern: union of the columns of the fine rows in each P^T row
      std::vector<std::vector<int32_t>> rows(nn);
      parallel_for(nn, [&](int I) {
        auto& r = rows[I];
        for (int q = tp[I]; q < tp[I + 1]; ++q) {
          const int i = trow[q];
          r.insert(r.end(), A.ci.begin() + A.rp[i], A.ci.begin() + A.rp[i + 1]);
        }
      });
      HPat Rp = finish(rows);
      upload_csr(L.R, Rp);
    }
    L.ptv.alloc(std::max<size_t>(tidx.size(), 1));
    L.ptvf.alloc(std::max<size_t>(tidx.size(), 1));
    L.P.vf.alloc(std::max<long long>(L.P.nnz, 1));
    // AP = A P pattern, then next-level pattern P^T (AP)
    HPat AP;
    {
      std::vector<std::vector<int32_t>> rows(n);
      parallel_for(n, [&](int i) {
        auto& r = rows[i];
        for (int k = A.rp[i]; k < A.rp[i + 1]; ++k) {
          int j = A.ci[k];
          for (int m = Pp.rp[j]; m < Pp.rp[j + 1]; ++m) r.push_back(Pp.ci[m]);
        }
      });
      AP = finish(rows);
    }
    upload_csr(L.AP, AP);
    HPat An;
    {
      std::vector<std::vector<int32_t>> rows(nn);
      parallel_for(nn, [&](int I) {
        auto& r = rows[I];
        for (int q = tp[I]; q < tp[I + 1]; ++q) {
          int i = trow[q];
          r.insert(r.end(), AP.ci.begin() + AP.rp[i], AP.ci.begin() + AP.rp[i + 1]);
        }
      });
      An = finish(rows);
    }
    if (getenv("HC_AMG_VERBOSE"))
      fprintf(stderr, "amg field %d level %d: n=%d active=%d nnz=%zu P.nnz=%zu -> next n=%d nnz=%zu\n",
              field, level, n, active, A.ci.size(), Pp.ci.size(), nn, An.ci.size());
    A = std::move(An);
    G = std::move(Gn);
    bx = nbx; by = nby; bz = nbz; ph = nph;
    sx = nx2; sy = ny2; sz = nz2;
    ++level;
  }
  for (size_t l = 1; l < B.levels.size(); ++l) {
    AmgLevel& L = B.levels[l];
    int m = std::max(L.n, 1);
    L.x.alloc(m); L.x2.alloc(m); L.b.alloc(m); L.res.alloc(m); L.acc.alloc(m); L.dinvc.alloc(m);
  }
  int nc = B.levels.back().n;
  if (nc > HC_COARSE_CAP)
    throw Error(HC_ERR_CUDA, "aggregation hierarchy left " + std::to_string(nc) +
                                 " coarsest unknowns (limit " + std::to_string(HC_COARSE_CAP) + ")");
  B.dense.alloc((size_t)std::max(nc, 1) * std::max(nc, 1));
  B.dense_inv.alloc((size_t)std::max(nc, 1) * std::max(nc, 1));
  if (nc > HC_COARSE_MAX) {   // blocked Gauss-Jordan work space: [A | I], a column panel, a row panel, a pivot block
    B.gj_aug.alloc((size_t)nc * 2 * nc);
    B.gj_col.alloc((size_t)nc * GJ_B);
    B.gj_row.alloc((size_t)GJ_B * 2 * nc);
    B.gj_piv.alloc((size_t)2 * GJ_B * GJ_B);
  }
  // cluster-fused tail of the cycle: the deepest run of CSR levels that are all small
  // (and plain V-cycle levels), if it spans at least two levels
  const int nl = (int)B.levels.size();
  int from = nl - 1;
  while (from - 1 >= 1) {
    const AmgLevel& L = B.levels[from - 1];
    const bool wcyc = cfg.gamma > 1 && from - 1 >= cfg.wmin && from - 1 <= cfg.wdepth;
    if (L.n > cfg.fuse_rows || L.A.nnz > cfg.fuse_nnz || wcyc) break;
    --from;
  }
  B.fuse_from = (cfg.fuse_rows > 0 && from <= nl - 2) ? from : -1;
  if (B.fuse_from >= 1) {
    std::vector<CoarseLev> h;
    for (int l = B.fuse_from; l < nl; ++l) {
      AmgLevel& L = B.levels[l];
      CoarseLev c{};
      c.n = L.n;
      c.rp = L.A.rp.p; c.ci = L.A.ci.p;
      c.vf = cfg.fp32_coarse ? L.A.vf.p : nullptr;
      c.vd = L.A.v.p;
      c.dinv = L.dinvc.p;
      c.b = L.b.p; c.x = L.x.p; c.x2 = L.x2.p; c.res = L.res.p;
      c.tentative = L.P.nnz == (long long)L.n;
      c.parent = L.parent.p;
      c.prp = L.P.rp.p; c.pci = L.P.ci.p; c.pv = L.P.v.p;
      c.pt_ptr = L.pt_ptr.p; c.pt_row = L.pt_row.p; c.ptv = L.ptv.p;
      h.push_back(c);
    }
    B.clev.alloc(h.size());
    HC_CUDA(cudaMemcpy(B.clev.p, h.data(), h.size() * sizeof(CoarseLev), cudaMemcpyHostToDevice));
  }
}

Amg* build_amg(const Operator& op) {
  long long nvox = op.P.nvox;
  std::vector<uint8_t> lab(nvox);
  HC_CUDA(cudaMemcpy(lab.data(), op.labels.p, nvox, cudaMemcpyDeviceToHost));
  auto amg = std::make_unique<Amg>();
  if (const char* e = getenv("HC_AMG_NU")) amg->nu = amg->nu_c = atoi(e);
  if (const char* e = getenv("HC_AMG_NU_C")) amg->nu_c = atoi(e);
  if (const char* e = getenv("HC_AMG_SA_C")) amg->sa_levels_c = atoi(e);
  if (const char* e = getenv("HC_AMG_OMEGA")) amg->omega = atof(e);
  amg->w_pre = amg->w_post0 = amg->w_post1 = amg->wf_pre = amg->wf_post = amg->omega;
  if (const char* e = getenv("HC_AMG_W_PRE")) amg->w_pre = atof(e);
  if (const char* e = getenv("HC_AMG_W_POST0")) amg->w_post0 = atof(e);
  if (const char* e = getenv("HC_AMG_W_POST1")) amg->w_post1 = atof(e);
  if (const char* e = getenv("HC_AMG_WF_PRE")) amg->wf_pre = atof(e);
  if (const char* e = getenv("HC_AMG_WF_POST")) amg->wf_post = atof(e);
  amg->wf_post1 = amg->omega;
  if (const char* e = getenv("HC_AMG_WF_POST1")) amg->wf_post1 = atof(e);
  if (const char* e = getenv("HC_AMG_OMEGA_P")) amg->omega_p = atof(e);
  if (const char* e = getenv("HC_AMG_SA_LEVELS")) amg->sa_levels = atoi(e);
  if (const char* e = getenv("HC_AMG_SA_ROWS")) amg->sa_rows = atoi(e);
  if (const char* e = getenv("HC_AMG_SA_ROWS_MIN")) amg->sa_rows_min = atoi(e);
  if (const char* e = getenv("HC_AMG_SA_ANY")) amg->sa_any = atoi(e);
  if (const char* e = getenv("HC_AMG_ALPHA")) amg->alpha = atof(e);
  if (const char* e = getenv("HC_AMG_COARSE_MAX")) amg->coarse_max = atoi(e);
  if (const char* e = getenv("HC_AMG_GAMMA")) amg->gamma = atoi(e);
  if (const char* e = getenv("HC_AMG_WDEPTH")) amg->wdepth = atoi(e);
  if (const char* e = getenv("HC_AMG_WMIN")) amg->wmin = atoi(e);
  if (const char* e = getenv("HC_GRAPHS")) amg->use_graphs = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_REFRESH")) amg->refresh = atoi(e);
  if (const char* e = getenv("HC_AMG_FP32")) amg->fp32_coarse = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_CF")) amg->coarsen = std::max(2, atoi(e));
  if (const char* e = getenv("HC_AMG_REFRESH_SOLVES")) amg->refresh_solves = std::max(1, atoi(e));
  if (const char* e = getenv("HC_AMG_FUSE_ROWS")) amg->fuse_rows = atoi(e);
  if (const char* e = getenv("HC_AMG_FUSE_NNZ")) amg->fuse_nnz = atoll(e);
  if (const char* e = getenv("HC_AMG_FUSE_RESTRICT")) amg->fuse_restrict = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_FUSE_RESTRICT_SA")) amg->fuse_restrict_sa = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_PACK")) amg->pack = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_SKIP_PLANES")) amg->skip_planes = atoi(e) != 0;
  if (const char* e = getenv("HC_AMG_SPARSIFY")) amg->sparsify = atof(e);
  if (const char* e = getenv("HC_AMG_SPARSIFY_AVG")) amg->sparsify_avg = atof(e);
  if (const char* e = getenv("HC_AMG_SPARSIFY_ROWS")) amg->sparsify_min_rows = atoi(e);
  if (const char* e = getenv("HC_AMG_SELL")) amg->sell_max_avg = atoi(e);
  if (const char* e = getenv("HC_AMG_SA_FILTER")) amg->sa_filter = atoi(e);
  if (const char* e = getenv("HC_AMG_SELL_ROWS")) amg->sell_min_rows = atoi(e);
  if (const char* e = getenv("HC_AMG_SELL_LANE")) amg->sell_lane_nnz = atof(e);
  if (const char* e = getenv("HC_AMG_SELL_T")) amg->sell_force_t = atoi(e);
  auto t0 = std::chrono::steady_clock::now();
  for (int f = 0; f < 2; ++f) {
    amg->blk[f].nu = amg->nu;
    amg->blk[f].nu_c = amg->blk[f].pre_c = amg->blk[f].post_c = amg->nu_c;
  }
  if (const char* e = getenv("HC_AMG_PRE_C"))
    for (auto& b : amg->blk) b.pre_c = atoi(e);
  if (const char* e = getenv("HC_AMG_POST_C"))
    for (auto& b : amg->blk) b.post_c = atoi(e);
  if (const char* e = getenv("HC_AMG_NU_C0")) amg->blk[0].nu = atoi(e);
  if (const char* e = getenv("HC_AMG_NU_C_C0")) amg->blk[0].nu_c = amg->blk[0].pre_c = amg->blk[0].post_c = atoi(e);
  build_block(op, lab, 0, *amg, amg->blk[0]);
  build_block(op, lab, 1, *amg, amg->blk[1]);
  if (getenv("HC_AMG_VERBOSE"))
    fprintf(stderr, "amg setup %.3f s\n",
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  for (int f = 0; f < 2; ++f) {
    amg->rs[f].alloc(nvox);
    amg->ea[f].alloc(nvox);
    amg->eb[f].alloc(nvox);
    // (zeroed: the c-block sweeps skip the planes without c rows and rely on zeros there)
    HC_CUDA(cudaMemset(amg->rs[f].p, 0, nvox * sizeof(double)));
    HC_CUDA(cudaMemset(amg->ea[f].p, 0, nvox * sizeof(double)));
    HC_CUDA(cudaMemset(amg->eb[f].p, 0, nvox * sizeof(double)));
  }
  amg->res.alloc(nvox);
  amg->rc2.alloc(nvox);
  HC_CUDA(cudaMemset(amg->res.p, 0, nvox * sizeof(double)));
  HC_CUDA(cudaMemset(amg->rc2.p, 0, nvox * sizeof(double)));
  if (const char* e = getenv("HC_AMG_BDIAG")) amg->bdiag = atoi(e) != 0;
  if (amg->bdiag) {
    amg->res_c.alloc(nvox);
    HC_CUDA(cudaMemset(amg->res_c.p, 0, nvox * sizeof(double)));
    HC_CUDA(cudaStreamCreateWithFlags(&amg->side, cudaStreamNonBlocking));
    HC_CUDA(cudaEventCreateWithFlags(&amg->ev_fork, cudaEventDisableTiming));
    HC_CUDA(cudaEventCreateWithFlags(&amg->ev_join, cudaEventDisableTiming));
  }
  return amg.release();
}

// Numeric setup for the current linearization (op.if_coef) and dt.
// Decide the sparsified sweep patterns of a block (AmgLevel::As) from the level operators'
// current values: eager, once, at the block's first numeric setup.  Levels handled by the
// cluster-fused coarse cycle keep their full operators.
static void sparsify_block(const Amg& A, AmgBlock& B, cudaStream_t s) {
  HC_CUDA(cudaStreamSynchronize(s));
  const size_t lend = B.fuse_from >= 1 ? (size_t)B.fuse_from : B.levels.size() - 1;
  for (size_t l = 1; l < lend && l + 1 < B.levels.size(); ++l) {
    AmgLevel& L = B.levels[l];
    if (!L.A.pk_ok || L.n < A.sparsify_min_rows || (double)L.A.nnz / L.n <= A.sparsify_avg) continue;
    std::vector<int32_t> rp(L.n + 1), ci(L.A.nnz);
    std::vector<double> v(L.A.nnz);
    HC_CUDA(cudaMemcpy(rp.data(), L.A.rp.p, rp.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(ci.data(), L.A.ci.p, ci.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(v.data(), L.A.v.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<uint8_t> keep(L.A.nnz, 0);
    HPat sp;
    sp.rp.assign(L.n + 1, 0);
    for (int i = 0; i < L.n; ++i) {
      double aii = 0.0;
      for (int q = rp[i]; q < rp[i + 1]; ++q)
        if (ci[q] == i) aii = std::fabs(v[q]);
      int cnt = 0;
      for (int q = rp[i]; q < rp[i + 1]; ++q)
        if (ci[q] == i || std::fabs(v[q]) >= A.sparsify * aii) {
          keep[q] = 1;
          ++cnt;
        }
      sp.rp[i + 1] = sp.rp[i] + cnt;
    }
    sp.ci.resize(sp.rp[L.n]);
    for (int i = 0, qs = 0; i < L.n; ++i)
      for (int q = rp[i]; q < rp[i + 1]; ++q)
        if (keep[q]) sp.ci[qs++] = ci[q];
    if (sp.ci.size() * 10 > ci.size() * 9) continue;   // under 10 % to drop: not worth a second copy
    Csr& S = L.As;
    S.n = L.n;
    S.nnz = (long long)sp.ci.size();
    upload(S.rp, sp.rp);
    upload(S.ci, sp.ci);
    build_packed(S, sp);
    if (!S.pk_ok) continue;
    if (A.sell_max_avg > 0) {
      const double avg = (double)sp.ci.size() / L.n;
      int T = 1;
      while (T < 32 && avg / T > A.sell_lane_nnz) T *= 2;
      if (A.sell_force_t) T = A.sell_force_t;
      if ((long long)L.n * T >= A.sell_min_rows && avg <= A.sell_max_avg) build_sell(S, sp, T);
    }
    upload(L.sp_keep, keep);
    L.sp_ok = true;
    if (getenv("HC_AMG_VERBOSE"))
      fprintf(stderr, "amg field %d level %zu: sweeps on %zu of %zu entries (drop tolerance %g)\n", B.field, l,
              sp.ci.size(), ci.size(), A.sparsify);
  }
}

void amg_update(Operator& op, double inv_dt, int blocks, cudaStream_t s) {
  Amg& A = *op.amg;
  for (int f = 0; f < 2; ++f) {
    if (!(blocks & (1 << f))) continue;
    AmgBlock& B = A.blk[f];
    AmgLevel& L0 = B.levels[0];
    launch(k_assemble0, vox_grid(op.P), vox_block(), 0, s, op.P, f, op.labels.p, op.if_rank.p, op.if_dir.p,
                                                op.if_solid.p, op.if_kind.p, op.if_coef.p, op.n_if,
                                                inv_dt, L0.A.rp.p, L0.A.ci.p, L0.A.v.p, L0.dinv.p); HC_COUNT();
    for (size_t l = 0; l + 1 < B.levels.size(); ++l) {
      AmgLevel& L = B.levels[l];
      AmgLevel& U = B.levels[l + 1];
      if (l > 0) {
        launch(k_dinv, nblk(L.n), TPB, 0, s, L.n, L.A.rp.p, L.A.ci.p, L.A.v.p, L.dinv.p, L.dinvc.p); HC_COUNT();
      }
      launch(k_smooth_P, nblk(L.n), TPB, 0, s, L.n, (int)L.smoothed, A.omega_p, L.A.rp.p, L.A.ci.p,
                                           L.A.v.p, L.dinv.p, L.parent.p, L.P.rp.p, L.P.ci.p,
                                           L.P.v.p); HC_COUNT();
      launch(k_gather_ptv, nblk((long long)L.P.nnz), TPB, 0, s, (long long)L.P.nnz, L.pt_idx.p, L.P.v.p,
                                                           L.ptv.p); HC_COUNT();
      if (A.fp32_coarse && L.P.nnz) {   // fp32 transfer values for the cycle (restriction / prolongation)
        launch(k_to_float, nblk(L.P.nnz), TPB, 0, s, (long long)L.P.nnz, (const double*)L.ptv.p, L.ptvf.p); HC_COUNT();
        launch(k_to_float, nblk(L.P.nnz), TPB, 0, s, (long long)L.P.nnz, (const double*)L.P.v.p, L.P.vf.p); HC_COUNT();
      }
      launch(k_ap_w, nblk(32LL * L.n), TPB, 0, s, L.n, L.A.rp.p, L.A.ci.p, L.A.v.p, L.P.rp.p, L.P.ci.p, L.P.v.p,
                                     L.AP.rp.p, L.AP.ci.p, L.AP.v.p); HC_COUNT();
      launch(k_ptap_w, nblk(32LL * U.n), TPB, 0, s, U.n, L.pt_ptr.p, L.pt_row.p, L.pt_idx.p, L.P.v.p,
                                            L.AP.rp.p, L.AP.ci.p, L.AP.v.p, U.A.rp.p, U.A.ci.p,
                                            U.A.v.p); HC_COUNT();
    }
    if (!B.sp_done) {
      // the sweep patterns are fixed at the block's first numeric setup, which must be an
      // eager one (the solver runs one before it captures its graphs); a block first set up
      // inside a capture keeps its full operators for good
      B.sp_done = true;
      if (!op.capturing && A.sparsify > 0.0 && A.pack && A.fp32_coarse) sparsify_block(A, B, s);
    }
    for (size_t l = 1; l < B.levels.size(); ++l) {
      AmgLevel& L = B.levels[l];
      if (A.fp32_coarse && L.A.nnz) {
        launch(k_to_float, nblk(L.A.nnz), TPB, 0, s, L.A.nnz, L.A.v.p, L.A.vf.p); HC_COUNT();
        if (L.A.sl_n) {
          launch(k_sell_gather, nblk(L.A.sl_nnz), TPB, 0, s, L.A.sl_nnz, L.A.sl_map.p, L.A.vf.p, L.A.sl_vf.p);
          HC_COUNT();
        }
        if (L.sp_ok) {
          Csr& S = L.As;
          launch(k_pack_rows_sp, nblk(L.n), TPB, 0, s, L.n, L.A.rp.p, L.A.ci.p, (const double*)L.A.v.p,
                 (const uint8_t*)L.sp_keep.p, S.rp.p, (const uint16_t*)S.pk_off.p, S.pk.p, S.pk_diag.p);
          HC_COUNT();
          if (S.sl_n && S.sl_base.n) {
            launch(k_sell_pack, nblk(S.sl_nnz), TPB, 0, s, S.sl_nnz, S.sl_map.p, (const uint16_t*)S.sl_off.p,
                   (const uint32_t*)S.pk.p, S.sl_pk.p);
            HC_COUNT();
          }
        } else if (L.A.pk_ok) {
          launch(k_pack_rows, nblk(L.n), TPB, 0, s, L.n, L.A.rp.p, L.A.ci.p, (const double*)L.A.v.p,
                 (const uint16_t*)L.A.pk_off.p, L.A.pk.p, L.A.pk_diag.p);
          HC_COUNT();
          if (L.A.sl_n && L.A.sl_base.n) {
            launch(k_sell_pack, nblk(L.A.sl_nnz), TPB, 0, s, L.A.sl_nnz, L.A.sl_map.p,
                   (const uint16_t*)L.A.sl_off.p, (const uint32_t*)L.A.pk.p, L.A.sl_pk.p);
            HC_COUNT();
          }
        }
      }
      if (L.R.nnz && l + 1 < B.levels.size()) {
        const AmgLevel& U = B.levels[l + 1];
        launch(k_pta_w, nblk(32LL * U.n), TPB, 0, s, U.n, L.pt_ptr.p, L.pt_row.p, L.pt_idx.p,
               (const double*)L.P.v.p, L.A.rp.p, L.A.ci.p, L.A.v.p, L.R.rp.p, L.R.ci.p, L.R.v.p); HC_COUNT();
        if (A.fp32_coarse) {
          launch(k_to_float, nblk(L.R.nnz), TPB, 0, s, L.R.nnz, L.R.v.p, L.R.vf.p); HC_COUNT();
        }
      }
    }
    AmgLevel& C = B.levels.back();
    if (B.levels.size() > 1) {
      launch(k_dinv, nblk(C.n), TPB, 0, s, C.n, C.A.rp.p, C.A.ci.p, C.A.v.p, C.dinv.p, C.dinvc.p); HC_COUNT();
    }
    launch(k_dense_from_csr, nblk(C.n), TPB, 0, s, C.n, C.A.rp.p, C.A.ci.p, C.A.v.p, B.dense.p); HC_COUNT();
    size_t smem = (size_t)C.n * C.n * sizeof(double) + (size_t)C.n * sizeof(int);
    static bool attr = false;
    if (!attr) {
      HC_CUDA(cudaFuncSetAttribute(k_dense_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((size_t)HC_COARSE_MAX * HC_COARSE_MAX * 8 + HC_COARSE_MAX * 4)));
      attr = true;
    }
    if (C.n <= HC_COARSE_MAX) {
      launch(k_dense_inverse, 1, 256, smem, s, C.n, B.dense.p, B.dense_inv.p); HC_COUNT();
    } else {
      const int n = C.n;
      double* G = B.gj_aug.p;
      double* piv = B.gj_piv.p;
      double* pinv = piv + GJ_B * GJ_B;
      launch(k_gj_init, nblk(2LL * n * n), TPB, 0, s, n, (const double*)B.dense.p, G); HC_COUNT();
      for (int k0 = 0; k0 < n; k0 += GJ_B) {
        const int bw = std::min(GJ_B, n - k0);
        // columns that hold anything but the untouched parts of [A | I] at this step
        const int j0 = k0, j1 = n + k0 + bw;
        launch(k_gj_col, nblk((long long)n * bw), TPB, 0, s, n, k0, bw, (const double*)G, B.gj_col.p, piv); HC_COUNT();
        launch(k_gj_pivot_inverse, 1, 256, 0, s, bw, (const double*)piv, pinv); HC_COUNT();
        // row panel R = D G[k rows]; every other row i -= G[i][k cols] R; then the panel itself
        launch(k_gj_gemm, dim3((j1 - j0 + GJ_TN - 1) / GJ_TN, 1), 256, 0, s, bw, bw, j0, j1, 2 * n, 1.0, (const double*)pinv,
               (const double*)(G + (long long)k0 * 2 * n), 0.0, B.gj_row.p, 0, 0); HC_COUNT();
        launch(k_gj_gemm, dim3((j1 - j0 + GJ_TN - 1) / GJ_TN, (n + GJ_TM - 1) / GJ_TM), 256, 0, s, n, bw, j0, j1, 2 * n, -1.0,
               (const double*)B.gj_col.p, (const double*)B.gj_row.p, 1.0, G, k0, bw); HC_COUNT();
        launch(k_gj_row, nblk((long long)bw * (j1 - j0)), TPB, 0, s, n, k0, bw, j0, j1, (const double*)B.gj_row.p, G); HC_COUNT();
      }
      launch(k_gj_out, nblk((long long)n * n), TPB, 0, s, n, (const double*)G, B.dense_inv.p); HC_COUNT();
    }
    HC_CHECK_LAUNCH();
  }
}

// ---- cluster-fused coarse cycle ----------------------------------------------------
// The levels below fuse_from (a few thousand unknowns, <= ~300 k nonzeros) are far too
// small to fill the GPU, so every sweep / restriction / prolongation there costs a
// launch for ~1 us of work.  One launch of a 16-CTA thread-block cluster runs that whole
// part of the V-cycle instead: rows spread over the cluster's 16 k threads (8 lanes per
// row), phases separated by barrier.cluster (release/acquire), vectors written by other
// CTAs read with ld.global.cg.  Same arithmetic as k_csr_x / k_restrict_v /
// k_dense_matvec / k_csr_prolong.
namespace {
constexpr int CC_THREADS = 1024;

template <int XM>
__device__ void cc_sweep(const CoarseLev& L, int gt, int gn, double w, double alpha, const CV* x,
                         const CV* xc, CV* y, int resid) {
  const int lane = gt & 7;
  // warp-uniform trip count (the 8-lane shuffles need all 32 lanes of the warp)
  for (int i0 = (gt >> 5) * 4; i0 < L.n; i0 += (gn >> 5) * 4) {
    const int i = i0 + ((gt & 31) >> 3);
    const bool ok = i < L.n;
    auto xin = [&](int j) -> double {
      if (XM == 0) return (double)__ldcg(x + j);
      if (XM == 1) return w * (double)L.dinv[j] * (double)__ldcg(L.b + j);
      return (double)__ldcg(x + j) + alpha * (double)__ldcg(xc + L.parent[j]);
    };
    double s = 0.0;
    if (ok)
      for (int k = L.rp[i] + lane; k < L.rp[i + 1]; k += 8)
        s += (L.vf ? (double)L.vf[k] : L.vd[k]) * xin(L.ci[k]);
    s += __shfl_down_sync(0xffffffffu, s, 4, 8);
    s += __shfl_down_sync(0xffffffffu, s, 2, 8);
    s += __shfl_down_sync(0xffffffffu, s, 1, 8);
    if (ok && lane == 0) {
      const double bi = __ldcg(L.b + i);
      y[i] = (CV)(resid ? bi - s : xin(i) + w * (double)L.dinv[i] * (bi - s));
    }
  }
}

__global__ void __launch_bounds__(CC_THREADS, 1)
k_coarse_cycle(const CoarseLev* __restrict__ levs, int nlev, const double* __restrict__ dense_inv,
               double w, double alpha, int nu) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  const int gt = (int)cl.block_rank() * blockDim.x + threadIdx.x;
  const int gn = (int)cl.num_blocks() * blockDim.x;
  __shared__ CV* xs[16];     // current / scratch iterate per level (uniform pointer swaps)
  __shared__ CV* x2s[16];
  if (threadIdx.x < nlev) {
    xs[threadIdx.x] = levs[threadIdx.x].x;
    x2s[threadIdx.x] = levs[threadIdx.x].x2;
  }
  __syncthreads();
  // down: pre-smoothing from the zero guess, residual, restriction
  for (int l = 0; l + 1 < nlev; ++l) {
    const CoarseLev L = levs[l];
    CV*& x = xs[l];
    CV*& x2 = x2s[l];
    if (nu >= 2) {
      cc_sweep<1>(L, gt, gn, w, 0.0, nullptr, nullptr, x, 0);
      cl.sync();
      for (int k = 2; k < nu; ++k) {
        cc_sweep<0>(L, gt, gn, w, 0.0, x, nullptr, x2, 0);
        cl.sync();
        if (threadIdx.x == 0) { CV* t = x; x = x2; x2 = t; }
        __syncthreads();
      }
      cc_sweep<0>(L, gt, gn, 0.0, 0.0, x, nullptr, L.res, 1);
    } else {
      for (int i = gt; i < L.n; i += gn) x[i] = (CV)(w * (double)L.dinv[i] * (double)__ldcg(L.b + i));
      cl.sync();
      cc_sweep<1>(L, gt, gn, w, 0.0, nullptr, nullptr, L.res, 1);
    }
    cl.sync();
    const CoarseLev U = levs[l + 1];
    const int lane = gt & 7;
    for (int I0 = (gt >> 5) * 4; I0 < U.n; I0 += (gn >> 5) * 4) {
      const int I = I0 + ((gt & 31) >> 3);
      double s = 0.0;
      if (I < U.n)
        for (int q = L.pt_ptr[I] + lane; q < L.pt_ptr[I + 1]; q += 8) s += L.ptv[q] * (double)__ldcg(L.res + L.pt_row[q]);
      s += __shfl_down_sync(0xffffffffu, s, 4, 8);
      s += __shfl_down_sync(0xffffffffu, s, 2, 8);
      s += __shfl_down_sync(0xffffffffu, s, 1, 8);
      if (I < U.n && lane == 0) U.b[I] = (CV)s;
    }
    cl.sync();
  }
  {  // coarsest: x = A^-1 b (explicit inverse), warp per row
    const CoarseLev C = levs[nlev - 1];
    const int lane = gt & 31;
    for (int row = gt >> 5; row < C.n; row += gn >> 5) {
      double s = 0.0;
      for (int j = lane; j < C.n; j += 32) s += dense_inv[row * C.n + j] * (double)__ldcg(C.b + j);
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) xs[nlev - 1][row] = (CV)s;
    }
    cl.sync();
  }
  // up: coarse correction (fused into the first post-sweep for tentative prolongators)
  for (int l = nlev - 2; l >= 0; --l) {
    const CoarseLev L = levs[l];
    CV*& x = xs[l];
    CV*& x2 = x2s[l];
    const CV* xc = xs[l + 1];
    int post = nu;
    if (L.tentative && post >= 1) {
      cc_sweep<2>(L, gt, gn, w, alpha, x, xc, x2, 0);
      cl.sync();
      if (threadIdx.x == 0) { CV* t = x; x = x2; x2 = t; }
      __syncthreads();
      --post;
    } else {
      for (int i = gt; i < L.n; i += gn) {
        double s = 0.0;
        for (int m = L.prp[i]; m < L.prp[i + 1]; ++m) s += L.pv[m] * (double)__ldcg(xc + L.pci[m]);
        x[i] = (CV)((double)__ldcg(x + i) + alpha * s);
      }
      cl.sync();
    }
    for (int k = 0; k < post; ++k) {
      cc_sweep<0>(L, gt, gn, w, 0.0, x, nullptr, x2, 0);
      cl.sync();
      if (threadIdx.x == 0) { CV* t = x; x = x2; x2 = t; }
      __syncthreads();
    }
  }
  // the caller reads the result from levels[fuse_from].x
  if (xs[0] != levs[0].x) {
    for (int i = gt; i < levs[0].n; i += gn) levs[0].x[i] = __ldcg(xs[0] + i);
  }
}
}  // namespace

static void coarse_cycle_launch(const Amg& A, AmgBlock& B, cudaStream_t s) {
  static int cluster = 0;
  if (!cluster) {
    cluster = 8;
    if (cudaFuncSetAttribute(k_coarse_cycle, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(CC_THREADS);
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = 16; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
      q.attrs = &at;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_coarse_cycle, &q) == cudaSuccess && n >= 1) cluster = 16;
    }
    cudaGetLastError();
    if (const char* e = getenv("HC_AMG_FUSE_CLUSTER")) cluster = atoi(e) >= 16 ? 16 : std::max(1, atoi(e));
  }
  static const int threads = getenv("HC_AMG_FUSE_THREADS") ? atoi(getenv("HC_AMG_FUSE_THREADS")) : CC_THREADS;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(threads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const int nlev = (int)B.levels.size() - B.fuse_from;
  HC_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_cycle, (const CoarseLev*)B.clev.p, nlev,
                             (const double*)B.dense_inv.p, A.omega, B.alpha, B.nu_c));
  HC_COUNT();
}

static void solve_level(const Amg& A, AmgBlock& B, size_t l, cudaStream_t s);

// y = x + w D^-1 (b - A x)  or  (resid) y = b - A x, with lanes-per-row from the density
static void csr_sweep(const Amg& A, const AmgLevel& L, double w, const CV* b, const CV* x,
                      CV* y, int resid, cudaStream_t s) {
  double avg = L.n ? (double)L.A.nnz / L.n : 0.0;
  const bool f32 = A.fp32_coarse;
  auto go = [&](auto vs_tag, auto* vals) {
    constexpr int VS = decltype(vs_tag)::value;
    using VT = std::remove_const_t<std::remove_pointer_t<decltype(vals)>>;
    launch(k_csr_jacobi_v<VS, VT>, nblk((long long)VS * L.n), TPB, 0, s, L.n, w, L.A.rp.p, L.A.ci.p, vals,
                                                                      L.dinvc.p, b, x, y, resid);
    HC_COUNT();
  };
  if (avg <= 12.0) {
    if (f32) go(std::integral_constant<int, 1>{}, (const float*)L.A.vf.p);
    else go(std::integral_constant<int, 1>{}, (const double*)L.A.v.p);
  } else if (avg <= 48.0) {
    if (f32) go(std::integral_constant<int, 8>{}, (const float*)L.A.vf.p);
    else go(std::integral_constant<int, 8>{}, (const double*)L.A.v.p);
  } else {
    if (f32) go(std::integral_constant<int, 32>{}, (const float*)L.A.vf.p);
    else go(std::integral_constant<int, 32>{}, (const double*)L.A.v.p);
  }
}

// generalized sweep launcher (see k_csr_x)
template <int XM>
static void csr_sweep_x(const Amg& A, const AmgLevel& L, double w, double alpha, const CV* b,
                        const CV* x, const int32_t* parent, const CV* xc, CV* y,
                        int resid, cudaStream_t s, CV* x0 = nullptr) {
  const Csr& S = L.sp_ok ? L.As : L.A;   // the sweeps' operator: sparsified copy where there is one
  if (A.fp32_coarse && S.sl_n && S.pk_ok && S.sl_base.n) {
    auto go = [&](auto t_tag) {
      constexpr int T = decltype(t_tag)::value;
      const long long threads = ((long long)L.n + 32 / T - 1) / (32 / T) * 32;
      launch(k_sell_xp<T, XM>, nblk(threads), TPB, 0, s, L.n, w, alpha, S.sl_ptr.p, S.sl_base.p,
             (const uint32_t*)S.sl_pk.p, (const float*)S.pk_diag.p, L.dinvc.p, b, x, parent, xc, y, resid, x0);
      HC_COUNT();
    };
    switch (S.sl_t) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 4: go(std::integral_constant<int, 4>{}); break;
      case 8: go(std::integral_constant<int, 8>{}); break;
      case 16: go(std::integral_constant<int, 16>{}); break;
      default: go(std::integral_constant<int, 32>{}); break;
    }
    return;
  }
  if (A.fp32_coarse && L.A.sl_n && !L.sp_ok) {
    auto go = [&](auto t_tag) {
      constexpr int T = decltype(t_tag)::value;
      const long long threads = ((long long)L.n + 32 / T - 1) / (32 / T) * 32;
      launch(k_sell_x<T, XM>, nblk(threads), TPB, 0, s, L.n, w, alpha, L.A.sl_ptr.p, L.A.sl_col.p,
             (const float*)L.A.sl_vf.p, L.dinvc.p, b, x, parent, xc, y, resid, x0);
      HC_COUNT();
    };
    switch (L.A.sl_t) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 4: go(std::integral_constant<int, 4>{}); break;
      case 8: go(std::integral_constant<int, 8>{}); break;
      case 16: go(std::integral_constant<int, 16>{}); break;
      default: go(std::integral_constant<int, 32>{}); break;
    }
    return;
  }
  double avg = L.n ? (double)S.nnz / L.n : 0.0;
  const int VSsel = avg <= 12.0 ? 1 : (avg <= 48.0 ? 8 : 32);
  if (A.fp32_coarse && S.pk_ok) {
    auto gop = [&](auto vs_tag) {
      constexpr int VS = decltype(vs_tag)::value;
      launch(k_csr_xp<VS, XM>, nblk((long long)VS * L.n), TPB, 0, s, L.n, w, alpha, S.rp.p, S.pk_base.p,
             (const uint32_t*)S.pk.p, (const float*)S.pk_diag.p, L.dinvc.p, b, x, parent, xc, y, resid, x0);
      HC_COUNT();
    };
    if (VSsel == 1) gop(std::integral_constant<int, 1>{});
    else if (VSsel == 8) gop(std::integral_constant<int, 8>{});
    else gop(std::integral_constant<int, 32>{});
    return;
  }
  auto go = [&](auto vs_tag, auto* vals) {
    constexpr int VS = decltype(vs_tag)::value;
    using VT = std::remove_const_t<std::remove_pointer_t<decltype(vals)>>;
    launch(k_csr_x<VS, VT, XM>, nblk((long long)VS * L.n), TPB, 0, s, 
        L.n, w, alpha, L.A.rp.p, L.A.ci.p, vals, L.dinvc.p, b, x, parent, xc, y, resid, x0);
    HC_COUNT();
  };
  const float* vf = L.A.vf.p;
  const double* vd = L.A.v.p;
  if (VSsel == 1) { if (A.fp32_coarse) go(std::integral_constant<int, 1>{}, vf); else go(std::integral_constant<int, 1>{}, vd); }
  else if (VSsel == 8) { if (A.fp32_coarse) go(std::integral_constant<int, 8>{}, vf); else go(std::integral_constant<int, 8>{}, vd); }
  else { if (A.fp32_coarse) go(std::integral_constant<int, 32>{}, vf); else go(std::integral_constant<int, 32>{}, vd); }
}

// one cycle at CSR level l >= 1: rhs in L.b, result in L.x
static void cycle_once(const Amg& A, AmgBlock& B, size_t l, cudaStream_t s) {
  AmgLevel& L = B.levels[l];
  AmgLevel& U = B.levels[l + 1];
  // per-sweep Jacobi weights (all A.omega unless set): two post sweeps with the reciprocals of
  // the degree-2 Chebyshev roots of [lmax / a, lmax] damp that interval by the Chebyshev
  // polynomial instead of (1 - w l)^2
  const double w = A.w_pre;
  auto wpost = [&](int k) { return k == 0 ? A.w_post0 : (k == 1 ? A.w_post1 : A.omega); };
  // pre-smoothing from a zero guess: the first sweep materialises x0 = w D^-1 b itself
  int pre = B.pre_c;
  if (pre >= 2) {
    csr_sweep_x<1>(A, L, w, 0.0, L.b.p, nullptr, nullptr, nullptr, L.x.p, 0, s);
    for (int k = 2; k < pre; ++k) {
      csr_sweep_x<0>(A, L, w, 0.0, L.b.p, L.x.p, nullptr, nullptr, L.x2.p, 0, s);
      std::swap(L.x.p, L.x2.p);
    }
  }
  if (pre >= 2 && L.R.nnz && !L.sp_ok) {
    // residual and restriction in one pass: U.b = P^T b - (P^T A) x
    const double avg = U.n ? (double)L.R.nnz / U.n : 0.0;
    auto go = [&](auto vs_tag, auto* vals) {
      constexpr int VS = decltype(vs_tag)::value;
      using VT = std::remove_const_t<std::remove_pointer_t<decltype(vals)>>;
      const VT* ptv = std::is_same<VT, float>::value ? (const VT*)(const void*)L.ptvf.p
                                                     : (const VT*)(const void*)L.ptv.p;
      launch(k_resid_restrict<VS, VT>, nblk((long long)VS * U.n), TPB, 0, s, U.n, L.pt_ptr.p, L.pt_row.p,
             L.R.rp.p, L.R.ci.p, vals, ptv, L.b.p, L.x.p, U.b.p);
      HC_COUNT();
    };
    if (A.fp32_coarse) {
      if (avg <= 48.0) go(std::integral_constant<int, 8>{}, (const float*)L.R.vf.p);
      else go(std::integral_constant<int, 32>{}, (const float*)L.R.vf.p);
    } else {
      if (avg <= 48.0) go(std::integral_constant<int, 8>{}, (const double*)L.R.v.p);
      else go(std::integral_constant<int, 32>{}, (const double*)L.R.v.p);
    }
  } else {
    if (pre >= 2) {
      csr_sweep_x<0>(A, L, 0.0, 0.0, L.b.p, L.x.p, nullptr, nullptr, L.res.p, 1, s);
    } else {
      // x0 = w D^-1 b and b - A x0 in one pass
      csr_sweep_x<1>(A, L, w, 0.0, L.b.p, nullptr, nullptr, nullptr, L.res.p, 1, s, L.x.p);
    }
    if (A.fp32_coarse)
      launch(k_restrict_v<float, CV>, nblk(8LL * U.n), TPB, 0, s, U.n, L.pt_ptr.p, L.pt_row.p,
             (const float*)L.ptvf.p, L.res.p, U.b.p);
    else
      launch(k_restrict_v<double, CV>, nblk(8LL * U.n), TPB, 0, s, U.n, L.pt_ptr.p, L.pt_row.p,
             (const double*)L.ptv.p, L.res.p, U.b.p);
    HC_COUNT();
  }
  solve_level(A, B, l + 1, s);
  const bool tentative = L.P.nnz == (long long)L.n;  // one prolongator entry per row
  int post = B.post_c, kp = 0;
  if (tentative && post >= 1) {
    // prolongation fused into the first post-sweep (P0 entries are all 1)
    csr_sweep_x<2>(A, L, wpost(kp++), B.alpha, L.b.p, L.x.p, L.parent.p, U.x.p, L.x2.p, 0, s);
    std::swap(L.x.p, L.x2.p);
    --post;
  } else {
    if (A.fp32_coarse)
      launch(k_csr_prolong<float>, nblk(L.n), TPB, 0, s, L.n, B.alpha, L.P.rp.p, L.P.ci.p, (const float*)L.P.vf.p, U.x.p,
             L.x.p);
    else
    launch(k_csr_prolong<double>, nblk(L.n), TPB, 0, s, L.n, B.alpha, L.P.rp.p, L.P.ci.p, (const double*)L.P.v.p, U.x.p,
                                            L.x.p); HC_COUNT();
  }
  for (int k = 0; k < post; ++k) {
    csr_sweep_x<0>(A, L, wpost(kp++), 0.0, L.b.p, L.x.p, nullptr, nullptr, L.x2.p, 0, s);
    std::swap(L.x.p, L.x2.p);
  }
}

// approximate solve at level l >= 1 (rhs L.b -> L.x): gamma cycles on the first
// wdepth levels, one below, dense LU at the coarsest level
static void solve_level(const Amg& A, AmgBlock& B, size_t l, cudaStream_t s) {
  if (B.fuse_from >= 1 && (int)l == B.fuse_from) {
    coarse_cycle_launch(A, B, s);
    return;
  }
  AmgLevel& L = B.levels[l];
  if (l + 1 == B.levels.size()) {
    launch(k_dense_matvec, nblk(L.n, 8), 256, 0, s, L.n, B.dense_inv.p, L.b.p, L.x.p); HC_COUNT();
    return;
  }
  cycle_once(A, B, l, s);
  int g = ((int)l >= A.wmin && (int)l <= A.wdepth) ? A.gamma : 1;
  for (int k = 1; k < g; ++k) {
    HC_CUDA(cudaMemcpyAsync(L.acc.p, L.x.p, L.n * sizeof(CV), cudaMemcpyDeviceToDevice, s));
    csr_sweep(A, L, 0.0, L.b.p, L.acc.p, L.res.p, 1, s);
    std::swap(L.b.p, L.res.p);
    cycle_once(A, B, l, s);
    std::swap(L.b.p, L.res.p);
    launch(k_vec_add, nblk(L.n), TPB, 0, s, L.n, L.acc.p, L.x.p); HC_COUNT();
  }
}

namespace {
__global__ void k_smooth0_s(long long n, double w, const double* __restrict__ dinv,
                            const double* __restrict__ r, double* __restrict__ e) {
  pdl_wait();
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v < n) e[v] = w * dinv[v] * r[v];
}
// the same into one component of a double2 vector (stride 2)
__global__ void k_smooth0_s2(long long n, double w, const double* __restrict__ dinv,
                             const double* __restrict__ r, double* __restrict__ e) {
  pdl_wait();
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v < n) e[2 * v] = w * dinv[v] * r[v];
}
template <class TV>
__global__ void k_prolong0_s(long long n, double alpha, const int32_t* __restrict__ prp,
                             const int32_t* __restrict__ pci, const TV* __restrict__ pv,
                             const CV* __restrict__ x1, double* __restrict__ e) {
  pdl_wait();
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  int p0 = prp[v], p1 = prp[v + 1];
  if (p0 == p1) return;
  double s = 0.0;
  for (int m = p0; m < p1; ++m) s += (double)pv[m] * x1[pci[m]];
  e[v] += alpha * s;
}
// T r split into scalar field right-hand sides
__global__ void k_split_T(DevParams P, const uint8_t* __restrict__ lab, const double2* __restrict__ r,
                          double* __restrict__ rc, double* __restrict__ rp) {
  pdl_wait();
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  double2 a = r[v];
  rc[v] = lab[v] == EL ? a.x - P.t_plus * a.y : a.x;
  rp[v] = a.y;
}
__global__ void k_merge_s(long long n, const double* __restrict__ ec, const double* __restrict__ ep,
                          double2* __restrict__ z) {
  pdl_wait();
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v < n) z[v] = make_double2(ec ? ec[v] : 0.0, ep[v]);
}
}  // namespace

// one V-cycle for block f on the fine grid, scalar vectors: e = M_f^{-1} r.
// Returns the buffer holding e (one of the block's two ping-pong vectors).
// dst (optional): the final sweep writes component f of that double2 vector instead
// (stride-2 output), and nullptr is returned
static double* vcycle_fine(Operator& op, int f, const double* r, double inv_dt, cudaStream_t s,
                           double2* dst = nullptr) {
  Amg& A = *op.amg;
  AmgBlock& B = A.blk[f];
  AmgLevel& L0 = B.levels[0];
  const long long nv = op.P.nvox;
  double w = A.wf_pre;   // weight of the sweep being launched (pre, then post)
  const int nb = nblk(nv);
  FineArgs F{op.labels.p, op.if_rank.p, op.if_vcoef.p, (long long)op.if_dir.n, op.inv_c.p,
             op.if_cslot.p, op.elz.p, nullptr, op.tp_off.p};
  if (A.skip_planes) F.cz = op.cz;
  const dim3 vg = vox_grid(op.P), vb = vox_block();
  double* e = A.ea[f].p;
  double* e2 = A.eb[f].p;
  double* res = (f == 0 && A.bdiag) ? A.res_c.p : A.res.p;
  auto sweep = [&](int epi, const double* in, double* out, int fl = 0) {
    if (f == 1) {
      if (epi == EP_SMOOTH0) fine_launch_op<SM_PHI, EP_SMOOTH0>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
      else if (epi == EP_SMOOTH) fine_launch_op<SM_PHI, EP_SMOOTH>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
      else fine_launch_op<SM_PHI, EP_RESID>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
    } else {
      if (epi == EP_SMOOTH0) fine_launch_op<SM_CONC, EP_SMOOTH0>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
      else if (epi == EP_SMOOTH) fine_launch_op<SM_CONC, EP_SMOOTH>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
      else fine_launch_op<SM_CONC, EP_RESID>(op, F, nullptr, in, r, L0.dinv.p, w, inv_dt, fl, nullptr, out, s);
    }
    HC_COUNT();
  };
  if (B.levels.size() == 1) {
    if (dst) {
      launch(k_smooth0_s2, nb, TPB, 0, s, nv, w, L0.dinv.p, r, reinterpret_cast<double*>(dst) + f); HC_COUNT();
      return nullptr;
    }
    launch(k_smooth0_s, nb, TPB, 0, s, nv, w, L0.dinv.p, r, e); HC_COUNT();
    return e;
  }
  AmgLevel& L1 = B.levels[1];
  if (B.nu >= 2) {
    sweep(EP_SMOOTH0, nullptr, e);          // e1 from the zero guess in one pass
    for (int k = 2; k < B.nu; ++k) {
      sweep(EP_SMOOTH, e, e2);
      std::swap(e, e2);
    }
  } else {
    // nu = 1: the zero-guess step e = w D^-1 r and the residual r - A e in one pass
    double2* e_out = reinterpret_cast<double2*>(e);
    if (f == 1)
      fine_launch_op<SM_PHI, EP_RESID0>(op, F, nullptr, nullptr, r, L0.dinv.p, w, inv_dt, 0, e_out, res, s);
    else
      fine_launch_op<SM_CONC, EP_RESID0>(op, F, nullptr, nullptr, r, L0.dinv.p, w, inv_dt, 0, e_out, res, s);
    HC_COUNT();
  }
  if (B.nu >= 2) sweep(EP_RESID, e, res);
  if (A.fp32_coarse)
    launch(k_restrict_v<float, double>, nblk(8LL * L1.n), TPB, 0, s, L1.n, L0.pt_ptr.p, L0.pt_row.p, (const float*)L0.ptvf.p,
           res, L1.b.p);
  else
  launch(k_restrict_v<double, double>, nblk(8LL * L1.n), TPB, 0, s, L1.n, L0.pt_ptr.p, L0.pt_row.p, (const double*)L0.ptv.p, res,
                                                L1.b.p); HC_COUNT();
  solve_level(A, B, 1, s);
  if (A.fp32_coarse)
    launch(k_prolong0_s<float>, nb, TPB, 0, s, nv, B.alpha, L0.P.rp.p, L0.P.ci.p, (const float*)L0.P.vf.p, L1.x.p, e);
  else
    launch(k_prolong0_s<double>, nb, TPB, 0, s, nv, B.alpha, L0.P.rp.p, L0.P.ci.p, (const double*)L0.P.v.p, L1.x.p, e);
  HC_COUNT();
  for (int k = 0; k < B.nu; ++k) {
    w = k == 0 ? A.wf_post : A.wf_post1;
    if (dst && k + 1 == B.nu) {
      sweep(EP_SMOOTH, e, reinterpret_cast<double*>(dst) + f, FL_OSTRIDE2);
      HC_CHECK_LAUNCH();
      return nullptr;
    }
    sweep(EP_SMOOTH, e, e2);
    std::swap(e, e2);
  }
  HC_CHECK_LAUNCH();
  return e;
}

// z = M^{-1} r for the full (c, phi) system; mode 0 full, 1 phi block only
static void amg_apply_impl(Operator& op, const double2* r, double2* z, double inv_dt, int mode,
                           cudaStream_t s, bool presplit) {
  Amg& A = *op.amg;
  const long long nv = op.P.nvox;
  const int nb = nblk(nv);
  if (!presplit) {
    launch(k_split_T, nb, TPB, 0, s, op.P, op.labels.p, r, A.rs[0].p, A.rs[1].p); HC_COUNT();
  }
  if (mode == 0 && A.bdiag) {
    // block Jacobi: fork the c-block V-cycle onto the side stream, join before the merge
    HC_CUDA(cudaEventRecord(A.ev_fork, s));
    HC_CUDA(cudaStreamWaitEvent(A.side, A.ev_fork, 0));
    // each block's final sweep writes its component of z (no merge pass)
    vcycle_fine(op, 0, A.rs[0].p, inv_dt, A.side, z);
    HC_CUDA(cudaEventRecord(A.ev_join, A.side));
    vcycle_fine(op, 1, A.rs[1].p, inv_dt, s, z);
    HC_CUDA(cudaStreamWaitEvent(s, A.ev_join, 0));
    HC_CHECK_LAUNCH();
    return;
  }
  double* ep = vcycle_fine(op, 1, A.rs[1].p, inv_dt, s);
  if (mode == 1) {
    launch(k_merge_s, nb, TPB, 0, s, nv, nullptr, ep, z); HC_COUNT();
    return;
  }
  // c-block right-hand side: T r_c - (T J)_cp e_phi
  FineArgs F{op.labels.p, op.if_rank.p, op.if_vcoef.p, (long long)op.if_dir.n, op.inv_c.p,
             op.if_cslot.p, op.elz.p, nullptr, op.tp_off.p};
  if (A.skip_planes) F.cz = op.cz;
  fine_launch_op<SM_CP, EP_RESID>(op, F, nullptr, ep, A.rs[0].p, nullptr, 0.0, inv_dt, 0,
                                  nullptr, A.rc2.p, s);
  HC_COUNT();
  double* ec = vcycle_fine(op, 0, A.rc2.p, inv_dt, s);
  launch(k_merge_s, nb, TPB, 0, s, nv, ec, ep, z); HC_COUNT();
  HC_CHECK_LAUNCH();
}

// The preconditioner is a fixed kernel sequence for fixed (r, z, mode, dt): it is
// captured once into a CUDA graph and replayed (the Galerkin values it reads
// live in device memory, so re-linearization does not invalidate the graph).
void amg_apply(Operator& op, const double2* r, double2* z, double inv_dt, int mode,
               cudaStream_t s, bool presplit) {
  Amg& A = *op.amg;
  if (!A.use_graphs || s == 0 || op.capturing) {
    amg_apply_impl(op, r, z, inv_dt, mode, s, presplit);
    return;
  }
  for (auto& g : A.graphs)
    if (g.r == r && g.z == z && g.mode == mode && g.inv_dt == inv_dt && g.presplit == presplit) {
      HC_CUDA(cudaGraphLaunch(g.exec, s));
      count_graph_launch(g.n_kernels);
      return;
    }
  AmgGraph g;
  g.r = r; g.z = z; g.mode = mode; g.inv_dt = inv_dt; g.presplit = presplit;
  unsigned long long c0 = t_launch_count;
  cudaGraph_t graph;
  HC_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  amg_apply_impl(op, r, z, inv_dt, mode, s, presplit);
  HC_CUDA(cudaStreamEndCapture(s, &graph));
  g.n_kernels = t_launch_count - c0;
  uncount(g.n_kernels);
  HC_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
  HC_CUDA(cudaGraphDestroy(graph));
  if (A.graphs.size() >= 16) {
    cudaGraphExecDestroy(A.graphs.front().exec);
    A.graphs.erase(A.graphs.begin());
  }
  A.graphs.push_back(g);
  HC_CUDA(cudaGraphLaunch(g.exec, s));
  count_graph_launch(g.n_kernels);
}

Amg::~Amg() {
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (side) cudaStreamDestroy(side);
}

}  // namespace hc
