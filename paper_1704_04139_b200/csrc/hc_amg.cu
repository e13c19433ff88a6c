// Field-split, phase-aware aggregation multigrid preconditioner.
//
// The reference factorizes the Newton Jacobian with SuperLU or ILU+LGMRES
// (fvm/newton.py:75-83).  On the device the Jacobian stays matrix-free and the
// linear solve is a Krylov method preconditioned by:
//   1. the row transform T (electrolyte c row -= t+ * phi row of the same voxel),
//      which cancels the migration and chemical-potential couplings exactly;
//   2. a block lower-triangular split of T J: phi block first, then c block;
//   3. one V-cycle per block of an unsmoothed-aggregation multigrid whose
//      aggregates are (2^l x 2^l x 2^l block, phase) pairs — aggregation never
//      mixes phases, so weakly coupled conductor clusters keep their own coarse
//      unknowns (their near-null constant modes survive coarsening).
// Level-1 Galerkin rows are gathered per coarse unknown from the matrix-free
// fine stencil (deterministic, no atomics); deeper levels are CSR.
#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>

#include "hc_amg.cuh"

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
  // binary search in [lo, hi)
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (col[mid] < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---- level-1 Galerkin rows gathered from the fine matrix-free operator ------
// field 1 (phi block, J_pp) or 0 (c block of T J incl. mass).  Also writes the
// fine-level inverse diagonal of every child voxel.
__global__ void k_galerkin1(DevParams P, int field, int n1, const int32_t* __restrict__ ch_ptr,
                            const int32_t* __restrict__ ch_vox, const uint8_t* __restrict__ lab,
                            const int32_t* __restrict__ agg1, const int32_t* __restrict__ if_rank,
                            const int32_t* __restrict__ if_dir, const int32_t* __restrict__ if_so,
                            const int8_t* __restrict__ if_kind, const double* __restrict__ coef,
                            long long n_if, double inv_dt, const int32_t* __restrict__ rowptr,
                            const int32_t* __restrict__ col, double* __restrict__ val,
                            double* __restrict__ fine_dinv) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n1) return;
  int r0 = rowptr[I], r1 = rowptr[I + 1];
  for (int k = r0; k < r1; ++k) val[k] = 0.0;
  int dpos = find_col(col, r0, r1, I);
  const double tp = P.t_plus;
  for (int q = ch_ptr[I]; q < ch_ptr[I + 1]; ++q) {
    long long v = ch_vox[q];
    int x = (int)(v % P.nx);
    long long t = v / P.nx;
    int y = (int)(t % P.ny), z = (int)(t / P.ny);
    uint8_t a = lab[v];
    double diag = 0.0;
    if (field == 0) diag += inv_dt;
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
      double off = 0.0;  // coupling A[v, nb]
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
          int f = if_dir[6LL * rk + d];
          double g = coef[2 * n_if + f];
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
          bool solid = if_so[f] == (int32_t)v;
          if (solid) {            // graphite c row: dv = ca vc_s + cb vc_e + ...
            if (if_kind[f] == IF_BV) { diag += ca; off = cb; has = true; }
          } else {                // electrolyte c row: -(1-t+) dv
            diag += -(1.0 - tp) * cb;
            if (if_kind[f] == IF_BV) { off = -(1.0 - tp) * ca; has = true; }
          }
        }
      }
      if (has) {
        int J = agg1[nb];
        if (J < 0) continue;
        if (J == I) val[dpos] += off;
        else val[find_col(col, r0, r1, J)] += off;
      }
    }
    val[dpos] += diag;
    fine_dinv[v] = diag != 0.0 ? 1.0 / diag : 0.0;
  }
}

// ---- level l -> l+1 Galerkin (unsmoothed aggregation, R = P^T) --------------
__global__ void k_galerkin_up(int n_up, const int32_t* __restrict__ ch_ptr,
                              const int32_t* __restrict__ ch, const int32_t* __restrict__ rp,
                              const int32_t* __restrict__ cl, const double* __restrict__ vl,
                              const int32_t* __restrict__ parent, const int32_t* __restrict__ rpu,
                              const int32_t* __restrict__ clu, double* __restrict__ vu) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n_up) return;
  int r0 = rpu[I], r1 = rpu[I + 1];
  for (int k = r0; k < r1; ++k) vu[k] = 0.0;
  for (int q = ch_ptr[I]; q < ch_ptr[I + 1]; ++q) {
    int i = ch[q];
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      int J = parent[cl[k]];
      vu[find_col(clu, r0, r1, J)] += vl[k];
    }
  }
}

__global__ void k_dinv(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cl,
                       const double* __restrict__ v, double* __restrict__ dinv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (cl[k] == i) d = v[k];
  dinv[i] = d != 0.0 ? 1.0 / d : 0.0;
}

// ---- coarsest level: dense LU with partial pivoting in one CTA --------------
__global__ void k_dense_from_csr(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cl,
                                 const double* __restrict__ v, double* __restrict__ A) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < n; ++j) A[(long long)i * n + j] = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) A[(long long)i * n + cl[k]] = v[k];
}

__global__ void k_dense_lu(int n, double* __restrict__ A, int* __restrict__ piv) {
  __shared__ double smax[1024];
  __shared__ int sidx[1024];
  int tid = threadIdx.x;
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = k;
    for (int i = k + tid; i < n; i += blockDim.x) {
      double a = fabs(A[(long long)i * n + k]);
      if (a > best) { best = a; bi = i; }
    }
    smax[tid] = best;
    sidx[tid] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if (tid < s) {
        if (smax[tid + s] > smax[tid] || (smax[tid + s] == smax[tid] && sidx[tid + s] < sidx[tid])) {
          smax[tid] = smax[tid + s];
          sidx[tid] = sidx[tid + s];
        }
      }
      __syncthreads();
    }
    int p = sidx[0];
    if (tid == 0) piv[k] = p;
    if (p != k)
      for (int j = tid; j < n; j += blockDim.x) {
        double t = A[(long long)k * n + j];
        A[(long long)k * n + j] = A[(long long)p * n + j];
        A[(long long)p * n + j] = t;
      }
    __syncthreads();
    double akk = A[(long long)k * n + k];
    double inv = akk != 0.0 ? 1.0 / akk : 0.0;
    for (int i = k + 1 + tid; i < n; i += blockDim.x) A[(long long)i * n + k] *= inv;
    __syncthreads();
    int m = n - k - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      int i = k + 1 + e / m, j = k + 1 + e % m;
      A[(long long)i * n + j] -= A[(long long)i * n + k] * A[(long long)k * n + j];
    }
    __syncthreads();
  }
}

__global__ void k_dense_solve(int n, const double* __restrict__ A, const int* __restrict__ piv,
                              const double* __restrict__ b, double* __restrict__ x) {
  extern __shared__ double y[];
  int tid = threadIdx.x;
  for (int i = tid; i < n; i += blockDim.x) y[i] = b[i];
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < n; ++k) {
      int p = piv[k];
      if (p != k) { double t = y[k]; y[k] = y[p]; y[p] = t; }
    }
  __syncthreads();
  for (int k = 0; k < n; ++k) {  // L (unit) forward
    double yk = y[k];
    for (int i = k + 1 + tid; i < n; i += blockDim.x) y[i] -= A[(long long)i * n + k] * yk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // U backward
    if (tid == 0) {
      double d = A[(long long)k * n + k];
      y[k] = d != 0.0 ? y[k] / d : 0.0;
    }
    __syncthreads();
    double yk = y[k];
    for (int i = tid; i < k; i += blockDim.x) y[i] -= A[(long long)i * n + k] * yk;
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) x[i] = y[i];
}

// ---- V-cycle kernels --------------------------------------------------------
__device__ __forceinline__ double fld(const double2& a, int f) { return f ? a.y : a.x; }

// e = w dinv r (field f), other component zero
__global__ void k_fine_smooth0(long long n, int f, double w, const double* __restrict__ dinv,
                               const double2* __restrict__ r, double2* __restrict__ e) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  double val = w * dinv[v] * fld(r[v], f);
  e[v] = f ? make_double2(0.0, val) : make_double2(val, 0.0);
}

// e += w dinv (r - t) on field f
__global__ void k_fine_smooth(long long n, int f, double w, const double* __restrict__ dinv,
                              const double2* __restrict__ r, const double2* __restrict__ t,
                              double2* __restrict__ e) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  double d = w * dinv[v] * (fld(r[v], f) - fld(t[v], f));
  if (f) e[v].y += d; else e[v].x += d;
}

// level-1 rhs: b1[I] = sum over children of (r - t)
__global__ void k_fine_restrict(int n1, int f, const int32_t* __restrict__ ch_ptr,
                                const int32_t* __restrict__ ch_vox, const double2* __restrict__ r,
                                const double2* __restrict__ t, double* __restrict__ b1) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n1) return;
  double s = 0.0;
  for (int q = ch_ptr[I]; q < ch_ptr[I + 1]; ++q) {
    int v = ch_vox[q];
    s += fld(r[v], f) - fld(t[v], f);
  }
  b1[I] = s;
}

__global__ void k_fine_prolong(long long n, int f, const int32_t* __restrict__ agg1,
                               const double* __restrict__ x1, double2* __restrict__ e) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  int I = agg1[v];
  if (I < 0) return;
  if (f) e[v].y += x1[I]; else e[v].x += x1[I];
}

__global__ void k_csr_smooth0(int n, double w, const double* __restrict__ dinv,
                              const double* __restrict__ b, double* __restrict__ x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = w * dinv[i] * b[i];
}

// y = x + w dinv (b - A x)
__global__ void k_csr_jacobi(int n, double w, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ cl, const double* __restrict__ v,
                             const double* __restrict__ dinv, const double* __restrict__ b,
                             const double* __restrict__ x, double* __restrict__ y) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = b[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k) s -= v[k] * x[cl[k]];
  y[i] = x[i] + w * dinv[i] * s;
}

// res = b - A x
__global__ void k_csr_resid(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ cl,
                            const double* __restrict__ v, const double* __restrict__ b,
                            const double* __restrict__ x, double* __restrict__ res) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = b[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k) s -= v[k] * x[cl[k]];
  res[i] = s;
}

__global__ void k_csr_restrict(int n_up, const int32_t* __restrict__ ch_ptr,
                               const int32_t* __restrict__ ch, const double* __restrict__ res,
                               double* __restrict__ b_up) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n_up) return;
  double s = 0.0;
  for (int q = ch_ptr[I]; q < ch_ptr[I + 1]; ++q) s += res[ch[q]];
  b_up[I] = s;
}

__global__ void k_csr_prolong(int n, const int32_t* __restrict__ parent,
                              const double* __restrict__ xu, double* __restrict__ x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += xu[parent[i]];
}

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h) {
  d.alloc(h.size());
  if (!h.empty()) HC_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}

}  // namespace

// ============================================================== host: pattern
// Build the aggregation hierarchy of one field from the host copy of the labels.
static void build_block(const Operator& op, const std::vector<uint8_t>& lab,
                        const std::vector<int32_t>& if_rank, const std::vector<int32_t>& if_dir,
                        const std::vector<int8_t>& if_kind, int field, int coarse_max,
                        AmgBlock& B) {
  const int nx = op.P.nx, ny = op.P.ny, nz = op.P.nz;
  const long long nxy = (long long)nx * ny, nvox = nxy * nz;
  B.field = field;
  auto in_field = [&](long long v) {
    uint8_t a = lab[v];
    if (field == 0) return a == GR || a == EL;
    return !((v / nxy) == nz - 1 && a == CC);
  };
  // ---- level 1 unknowns: (2x2x2 block, phase)
  int bx = (nx + 1) / 2, by = (ny + 1) / 2, bz = (nz + 1) / 2;
  long long nkeys = (long long)bx * by * bz * N_PHASES;
  std::vector<int32_t> keynum(nkeys, -1);
  for (long long v = 0; v < nvox; ++v) {
    if (!in_field(v)) continue;
    long long x = v % nx, y = (v / nx) % ny, z = v / nxy;
    long long key = (((z / 2) * by + y / 2) * bx + x / 2) * N_PHASES + lab[v];
    keynum[key] = 1;
  }
  int n1 = 0;
  std::vector<int32_t> ubx, uby, ubz, uph;
  for (long long k = 0; k < nkeys; ++k)
    if (keynum[k] >= 0) {
      keynum[k] = n1++;
      long long blk = k / N_PHASES;
      uph.push_back((int32_t)(k % N_PHASES));
      ubx.push_back((int32_t)(blk % bx));
      uby.push_back((int32_t)((blk / bx) % by));
      ubz.push_back((int32_t)(blk / ((long long)bx * by)));
    }
  std::vector<int32_t> agg1(nvox, -1);
  std::vector<int32_t> cnt(n1 + 1, 0);
  for (long long v = 0; v < nvox; ++v) {
    if (!in_field(v)) continue;
    long long x = v % nx, y = (v / nx) % ny, z = v / nxy;
    long long key = (((z / 2) * by + y / 2) * bx + x / 2) * N_PHASES + lab[v];
    agg1[v] = keynum[key];
    cnt[agg1[v] + 1]++;
  }
  std::vector<int32_t> chp(n1 + 1, 0), chv;
  for (int i = 0; i < n1; ++i) chp[i + 1] = chp[i] + cnt[i + 1];
  chv.resize(chp[n1]);
  {
    std::vector<int32_t> fill(chp.begin(), chp.end() - 1);
    for (long long v = 0; v < nvox; ++v)
      if (agg1[v] >= 0) chv[fill[agg1[v]]++] = (int32_t)v;
  }
  // level-1 pattern from fine couplings
  std::vector<std::vector<int32_t>> rows(n1);
  for (int I = 0; I < n1; ++I) rows[I].push_back(I);
  for (long long v = 0; v < nvox; ++v) {
    int I = agg1[v];
    if (I < 0) continue;
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
      int J = agg1[nb];
      if (J < 0 || J == I) continue;
      uint8_t b = lab[nb];
      uint8_t kd = kind_of(a, b);
      bool has;
      if (field == 1) has = kd == K_CONT || kd == K_CONTACT || kd == K_BV || kd == K_CE || kd == K_STRIP;
      else has = (kd == K_CONT) || (kd == K_BV);
      if (has) rows[I].push_back(J);
    }
  }
  auto finish_rows = [](std::vector<std::vector<int32_t>>& rws, std::vector<int32_t>& rp,
                        std::vector<int32_t>& cl) {
    rp.assign(rws.size() + 1, 0);
    cl.clear();
    for (size_t i = 0; i < rws.size(); ++i) {
      auto& r = rws[i];
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      rp[i + 1] = rp[i] + (int32_t)r.size();
      cl.insert(cl.end(), r.begin(), r.end());
    }
  };
  B.levels.clear();
  B.levels.emplace_back();
  {
    AmgLevel& L = B.levels.back();
    L.n = n1;
    std::vector<int32_t> rp, cl;
    finish_rows(rows, rp, cl);
    upload(L.rowptr, rp);
    upload(L.col, cl);
    L.val.alloc(std::max<size_t>(cl.size(), 1));
    upload(L.ch_ptr, chp);
    upload(L.ch, chv);
    L.nnz = (long long)cl.size();
    L.h_rowptr = rp;
    L.h_col = cl;
  }
  upload(B.agg1, agg1);
  B.fine_dinv.alloc(nvox);
  HC_CUDA(cudaMemset(B.fine_dinv.p, 0, nvox * sizeof(double)));
  // ---- deeper levels
  int sx = bx, sy = by, sz = bz;
  std::vector<int32_t> cbx = ubx, cby = uby, cbz = ubz, cph = uph;
  while (B.levels.back().n > coarse_max && (sx > 1 || sy > 1 || sz > 1)) {
    AmgLevel& L = B.levels.back();
    int nx2 = (sx + 1) / 2, ny2 = (sy + 1) / 2, nz2 = (sz + 1) / 2;
    long long nk = (long long)nx2 * ny2 * nz2 * N_PHASES;
    std::vector<int32_t> kn(nk, -1);
    std::vector<long long> keyof(L.n);
    for (int i = 0; i < L.n; ++i) {
      long long key = (((long long)(cbz[i] / 2) * ny2 + cby[i] / 2) * nx2 + cbx[i] / 2) * N_PHASES + cph[i];
      keyof[i] = key;
      kn[key] = 1;
    }
    int nu = 0;
    std::vector<int32_t> nbx, nby, nbz, nph;
    for (long long k = 0; k < nk; ++k)
      if (kn[k] >= 0) {
        kn[k] = nu++;
        long long blk = k / N_PHASES;
        nph.push_back((int32_t)(k % N_PHASES));
        nbx.push_back((int32_t)(blk % nx2));
        nby.push_back((int32_t)((blk / nx2) % ny2));
        nbz.push_back((int32_t)(blk / ((long long)nx2 * ny2)));
      }
    std::vector<int32_t> parent(L.n);
    for (int i = 0; i < L.n; ++i) parent[i] = kn[keyof[i]];
    std::vector<int32_t> c2(nu + 1, 0);
    for (int i = 0; i < L.n; ++i) c2[parent[i] + 1]++;
    std::vector<int32_t> cp(nu + 1, 0), cv(L.n);
    for (int i = 0; i < nu; ++i) cp[i + 1] = cp[i] + c2[i + 1];
    {
      std::vector<int32_t> fill(cp.begin(), cp.end() - 1);
      for (int i = 0; i < L.n; ++i) cv[fill[parent[i]]++] = i;
    }
    std::vector<std::vector<int32_t>> rws(nu);
    for (int i = 0; i < L.n; ++i)
      for (int k = L.h_rowptr[i]; k < L.h_rowptr[i + 1]; ++k)
        rws[parent[i]].push_back(parent[L.h_col[k]]);
    upload(L.parent, parent);
    AmgLevel U;
    U.n = nu;
    std::vector<int32_t> rp, cl;
    finish_rows(rws, rp, cl);
    upload(U.rowptr, rp);
    upload(U.col, cl);
    U.val.alloc(std::max<size_t>(cl.size(), 1));
    upload(U.ch_ptr, cp);
    upload(U.ch, cv);
    U.nnz = (long long)cl.size();
    U.h_rowptr = rp;
    U.h_col = cl;
    B.levels.push_back(std::move(U));
    sx = nx2; sy = ny2; sz = nz2;
    cbx = nbx; cby = nby; cbz = nbz; cph = nph;
  }
  for (auto& L : B.levels) {
    L.dinv.alloc(std::max(L.n, 1));
    L.x.alloc(std::max(L.n, 1));
    L.x2.alloc(std::max(L.n, 1));
    L.b.alloc(std::max(L.n, 1));
    L.res.alloc(std::max(L.n, 1));
    L.h_rowptr.clear(); L.h_rowptr.shrink_to_fit();
    L.h_col.clear(); L.h_col.shrink_to_fit();
  }
  int nc = B.levels.back().n;
  B.dense.alloc((size_t)nc * nc);
  B.piv.alloc(nc);
}

Amg* build_amg(const Operator& op) {
  long long nvox = op.P.nvox;
  std::vector<uint8_t> lab(nvox);
  HC_CUDA(cudaMemcpy(lab.data(), op.labels.p, nvox, cudaMemcpyDeviceToHost));
  std::vector<int32_t> if_rank(nvox), if_dir(op.if_dir.n);
  std::vector<int8_t> if_kind(op.n_if);
  HC_CUDA(cudaMemcpy(if_rank.data(), op.if_rank.p, nvox * 4, cudaMemcpyDeviceToHost));
  if (op.if_dir.n) HC_CUDA(cudaMemcpy(if_dir.data(), op.if_dir.p, op.if_dir.n * 4, cudaMemcpyDeviceToHost));
  if (op.n_if) HC_CUDA(cudaMemcpy(if_kind.data(), op.if_kind.p, op.n_if, cudaMemcpyDeviceToHost));
  auto amg = std::make_unique<Amg>();
  build_block(op, lab, if_rank, if_dir, if_kind, 0, amg->coarse_max, amg->blk[0]);
  build_block(op, lab, if_rank, if_dir, if_kind, 1, amg->coarse_max, amg->blk[1]);
  amg->t.alloc(nvox);
  amg->e.alloc(nvox);
  amg->zp.alloc(nvox);
  amg->rr.alloc(nvox);
  return amg.release();
}

// Numeric Galerkin products for the current linearization (op.if_coef) and dt.
void amg_update(Operator& op, double inv_dt, int blocks, cudaStream_t s) {
  Amg& A = *op.amg;
  for (int f = 0; f < 2; ++f) {
    if (!(blocks & (1 << f))) continue;
    AmgBlock& B = A.blk[f];
    AmgLevel& L1 = B.levels[0];
    k_galerkin1<<<nblk(L1.n), TPB, 0, s>>>(op.P, f, L1.n, L1.ch_ptr.p, L1.ch.p, op.labels.p,
                                           B.agg1.p, op.if_rank.p, op.if_dir.p, op.if_solid.p,
                                           op.if_kind.p, op.if_coef.p, op.n_if, inv_dt,
                                           L1.rowptr.p, L1.col.p, L1.val.p, B.fine_dinv.p);
    for (size_t l = 0; l + 1 < B.levels.size(); ++l) {
      AmgLevel& L = B.levels[l];
      AmgLevel& U = B.levels[l + 1];
      k_galerkin_up<<<nblk(U.n), TPB, 0, s>>>(U.n, U.ch_ptr.p, U.ch.p, L.rowptr.p, L.col.p,
                                              L.val.p, L.parent.p, U.rowptr.p, U.col.p, U.val.p);
    }
    for (auto& L : B.levels)
      k_dinv<<<nblk(L.n), TPB, 0, s>>>(L.n, L.rowptr.p, L.col.p, L.val.p, L.dinv.p);
    AmgLevel& C = B.levels.back();
    k_dense_from_csr<<<nblk(C.n), TPB, 0, s>>>(C.n, C.rowptr.p, C.col.p, C.val.p, B.dense.p);
    k_dense_lu<<<1, 1024, 0, s>>>(C.n, B.dense.p, B.piv.p);
    HC_CHECK_LAUNCH();
  }
}

// V-cycle on CSR levels l.. (level index into B.levels); rhs in L.b, result in L.x
static void vcycle_csr(AmgBlock& B, size_t l, int nu, double w, cudaStream_t s) {
  AmgLevel& L = B.levels[l];
  if (l + 1 == B.levels.size()) {
    k_dense_solve<<<1, 256, L.n * sizeof(double), s>>>(L.n, B.dense.p, B.piv.p, L.b.p, L.x.p);
    return;
  }
  AmgLevel& U = B.levels[l + 1];
  k_csr_smooth0<<<nblk(L.n), TPB, 0, s>>>(L.n, w, L.dinv.p, L.b.p, L.x.p);
  for (int k = 1; k < nu; ++k) {
    k_csr_jacobi<<<nblk(L.n), TPB, 0, s>>>(L.n, w, L.rowptr.p, L.col.p, L.val.p, L.dinv.p, L.b.p,
                                           L.x.p, L.x2.p);
    std::swap(L.x.p, L.x2.p);
  }
  k_csr_resid<<<nblk(L.n), TPB, 0, s>>>(L.n, L.rowptr.p, L.col.p, L.val.p, L.b.p, L.x.p, L.res.p);
  k_csr_restrict<<<nblk(U.n), TPB, 0, s>>>(U.n, U.ch_ptr.p, U.ch.p, L.res.p, U.b.p);
  vcycle_csr(B, l + 1, nu, w, s);
  k_csr_prolong<<<nblk(L.n), TPB, 0, s>>>(L.n, L.parent.p, U.x.p, L.x.p);
  for (int k = 0; k < nu; ++k) {
    k_csr_jacobi<<<nblk(L.n), TPB, 0, s>>>(L.n, w, L.rowptr.p, L.col.p, L.val.p, L.dinv.p, L.b.p,
                                           L.x.p, L.x2.p);
    std::swap(L.x.p, L.x2.p);
  }
}

// one V-cycle for field f on the fine grid: e = M_f^{-1} r (field component only)
static void vcycle_fine(Operator& op, int f, const double2* r, double2* e, double inv_dt,
                        cudaStream_t s) {
  Amg& A = *op.amg;
  AmgBlock& B = A.blk[f];
  AmgLevel& L1 = B.levels[0];
  const long long nv = op.P.nvox;
  const int flags = f ? 0 : (1 | 2);
  const double w = A.omega;
  k_fine_smooth0<<<nblk(nv), TPB, 0, s>>>(nv, f, w, B.fine_dinv.p, r, e);
  for (int k = 1; k < A.nu; ++k) {
    jvp_grid(op, e, inv_dt, flags, A.t.p, s);
    k_fine_smooth<<<nblk(nv), TPB, 0, s>>>(nv, f, w, B.fine_dinv.p, r, A.t.p, e);
  }
  jvp_grid(op, e, inv_dt, flags, A.t.p, s);
  k_fine_restrict<<<nblk(L1.n), TPB, 0, s>>>(L1.n, f, L1.ch_ptr.p, L1.ch.p, r, A.t.p, L1.b.p);
  vcycle_csr(B, 0, A.nu, w, s);
  k_fine_prolong<<<nblk(nv), TPB, 0, s>>>(nv, f, B.agg1.p, L1.x.p, e);
  for (int k = 0; k < A.nu; ++k) {
    jvp_grid(op, e, inv_dt, flags, A.t.p, s);
    k_fine_smooth<<<nblk(nv), TPB, 0, s>>>(nv, f, w, B.fine_dinv.p, r, A.t.p, e);
  }
  HC_CHECK_LAUNCH();
}

namespace {
// rr = T r : electrolyte c row -= t+ * phi row
__global__ void k_apply_T(DevParams P, const uint8_t* __restrict__ lab, const double2* __restrict__ r,
                          double2* __restrict__ out) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  double2 a = r[v];
  if (lab[v] == EL) a.x -= P.t_plus * a.y;
  out[v] = a;
}
// rc = rr.c - t.c (coupling), stored in .x of out; phi part from zp
__global__ void k_combine(long long n, const double2* __restrict__ rr, const double2* __restrict__ t,
                          double2* __restrict__ out) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  out[v] = make_double2(rr[v].x - t[v].x, 0.0);
}
__global__ void k_merge(long long n, const double2* __restrict__ zc, const double2* __restrict__ zp,
                        double2* __restrict__ z) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  z[v] = make_double2(zc[v].x, zp[v].y);
}
}  // namespace

// z = M^{-1} r for the full (c, phi) system; mode 0 full, 1 phi block only
void amg_apply(Operator& op, const double2* r, double2* z, double inv_dt, int mode,
               cudaStream_t s) {
  Amg& A = *op.amg;
  const long long nv = op.P.nvox;
  if (mode == 1) {
    vcycle_fine(op, 1, r, z, inv_dt, s);
    return;
  }
  k_apply_T<<<nblk(nv), TPB, 0, s>>>(op.P, op.labels.p, r, A.rr.p);
  vcycle_fine(op, 1, A.rr.p, A.zp.p, inv_dt, s);     // zp.y = phi correction, zp.x = 0
  jvp_grid(op, A.zp.p, inv_dt, 2, A.t.p, s);        // t.x = (T J)_cp zp
  k_combine<<<nblk(nv), TPB, 0, s>>>(nv, A.rr.p, A.t.p, A.e.p);
  vcycle_fine(op, 0, A.e.p, z, inv_dt, s);           // z.x = c correction
  k_merge<<<nblk(nv), TPB, 0, s>>>(nv, z, A.zp.p, z);
  HC_CHECK_LAUNCH();
}



}  // namespace hc
