// Fused matrix-free Jacobian stencil on the voxel grid (one pass, no atomics).
//
// One thread per voxel row.  All neighbour labels and values are loaded up front
// (clamped indices, masked) so every thread keeps 13+ independent loads in flight;
// the face coefficients are derived from the phase labels, and the linearized
// interface-face derivatives (Butler-Volmer, counter exchange, stripping) are read
// per (interface voxel, direction) through the voxel's interface rank (if_rank),
// so interface faces need no separate kernel and no atomics.
//
// Modes:
//   FULL: out2 = (J + mass) V  on double2 (c, phi) vectors, with the row transform
//         T and the 1/c terms selectable by flags (the Krylov operator);
//   PHI : scalar phi-block J_pp e (AMG fine level);
//   CONC: scalar c-block ((T J)_cc + mass) e (AMG fine level);
//   CP  : scalar coupling (T J)_cp e_phi on c rows (block-triangular preconditioner):
//         migration and phi-row terms cancel under T, only interface faces remain.
// Epilogues for PHI/CONC: SMOOTH y = e + w dinv (r - A e); RESID y = r - A e.
#pragma once

#include <algorithm>
#include <type_traits>

#include "hc_internal.cuh"

namespace hc {

enum { SM_FULL = 0, SM_PHI = 1, SM_CONC = 2, SM_CP = 3 };
enum { EP_STORE = 0, EP_SMOOTH = 1, EP_RESID = 2, EP_SMOOTH0 = 3 };  // SMOOTH0: first sweep from e0 = w D^-1 r

struct FineArgs {
  const uint8_t* lab;
  const int32_t* if_rank;
  const double* vcoef;    // interface derivatives per (interface voxel, direction): [3][nslot]
  long long nslot;        // 6 * number of interface voxels
  const double* w;        // gX / c per electrolyte voxel (FULL with flag 4)
};

template <int MODE, int EPI>
__global__ void __launch_bounds__(VX * VY)
k_fine_op(DevParams P, FineArgs F, const double2* __restrict__ V, const double* __restrict__ e,
          const double* __restrict__ r, const double* __restrict__ dinv, double omega,
          double inv_dt, int flags, double2* __restrict__ out2, double* __restrict__ out) {
  // face-coefficient tables in shared memory: branch-free faces, indexed a * 6 + b
  __shared__ double sP[36], sC[36], sM[36];
  __shared__ unsigned char sI[36];
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid < 36) {
    sP[tid] = P.gP[tid];
    sC[tid] = P.gC[tid];
    sM[tid] = P.gMig[tid];
    sI[tid] = P.ifc[tid];
  }
  __syncthreads();
  int x, y, z, v;
  if (!vox_index(P, x, y, z, v)) return;
  const uint8_t a = __ldg(F.lab + v);
  const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == GR || a == EL)
                                                         : !(z == P.nz - 1 && a == CC);
  if (!in_row) {
    if (MODE == SM_FULL) out2[v] = make_double2(0.0, 0.0);
    else out[v] = 0.0;
    return;
  }
  // out-of-domain neighbours alias the voxel itself: same phase, zero difference,
  // so they contribute nothing; grounded neighbours hold phi = 0 in every vector
  const int nxy = (int)P.nxy;
  int nb[6];
  nb[0] = x > 0 ? v - 1 : v;
  nb[1] = x + 1 < P.nx ? v + 1 : v;
  nb[2] = y > 0 ? v - P.nx : v;
  nb[3] = y + 1 < P.ny ? v + P.nx : v;
  nb[4] = z > 0 ? v - nxy : v;
  nb[5] = z + 1 < P.nz ? v + nxy : v;
  uint8_t lb[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) lb[d] = __ldg(F.lab + nb[d]);
  const int a6 = a * 6;
  const double tp = P.t_plus;
  double rc = 0.0, rp = 0.0;
  bool any_if = false;
#pragma unroll
  for (int d = 0; d < 6; ++d) any_if |= sI[a6 + lb[d]] != 0;
  if (MODE == SM_FULL) {
    const double2 Va = V[v];
    double2 Vb[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) Vb[d] = V[nb[d]];
    const bool one_c = (flags & 4) && a == EL;
    double wa = 0.0, wb[6];
    if (one_c) {
      wa = F.w[v];
#pragma unroll
      for (int d = 0; d < 6; ++d) wb[d] = F.w[nb[d]];
    }
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const int i = a6 + lb[d];
      const double dp = Va.y - Vb[d].y;
      rp += sP[i] * dp;
      rc += sC[i] * (Va.x - Vb[d].x) + sM[i] * dp;
      if (one_c && sM[i] != 0.0) {
        double dq = wa * Va.x - wb[d] * Vb[d].x;
        rp += dq;
        rc += tp * dq;
      }
    }
    if (any_if) {
      const int rk = __ldg(F.if_rank + v);
      const bool solid = a != EL;
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        const uint8_t b = lb[d];
        if (!sI[a6 + b]) continue;
        const long long f = 6LL * rk + d;
        const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f),
                     cg = __ldg(F.vcoef + 2 * F.nslot + f);
        const bool bv = a == GR || b == GR;
        const double2 vs = solid ? Va : Vb[d], ve = solid ? Vb[d] : Va;
        // dv = ca c_s + cb c_e + cg (phi_s - phi_e)  (ca = 0 unless BV)
        const double dv = (bv ? ca * vs.x : 0.0) + cb * ve.x + cg * (vs.y - ve.y);
        if (solid) {
          if (bv) rc += dv;
          rp += dv;
        } else {  // the row transform T is applied once below (rc -= t+ rp)
          rc -= dv;
          rp -= dv;
        }
      }
    }
    if ((flags & 1) && (a == GR || a == EL)) rc += Va.x * inv_dt;
    if ((flags & 2) && a == EL) rc -= tp * rp;
    if (flags & 8) rc = 0.0;
    out2[v] = make_double2(rc, rp);
    return;
  }
  const double ea = e[v];
  double eb[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) eb[d] = e[nb[d]];
  if (MODE == SM_PHI) {
#pragma unroll
    for (int d = 0; d < 6; ++d) rp += sP[a6 + lb[d]] * (ea - eb[d]);
  } else if (MODE == SM_CONC) {
#pragma unroll
    for (int d = 0; d < 6; ++d) rp += sC[a6 + lb[d]] * (ea - eb[d]);
    rp += inv_dt * ea;
  }
  if (any_if) {
    const int rk = __ldg(F.if_rank + v);
    const bool solid = a != EL;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      const uint8_t b = lb[d];
      if (!sI[a6 + b]) continue;
      const long long f = 6LL * rk + d;
      const bool bv = a == GR || b == GR;
      if (MODE == SM_PHI) {
        rp += __ldg(F.vcoef + 2 * F.nslot + f) * (ea - eb[d]);
      } else if (MODE == SM_CP) {
        const double cg = __ldg(F.vcoef + 2 * F.nslot + f);
        if (solid) {
          if (bv) rp += cg * (ea - eb[d]);
        } else {
          rp += (1.0 - tp) * cg * (ea - eb[d]);
        }
      } else {
        const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f);
        if (solid) {
          if (bv) rp += ca * ea + cb * eb[d];
        } else {
          rp -= (1.0 - tp) * ((bv ? ca * eb[d] : 0.0) + cb * ea);
        }
      }
    }
  }
  // SM_CP with EP_RESID: out = r - (T J)_cp e (the c-block right-hand side)
  if (EPI == EP_STORE) out[v] = rp;
  else if (EPI == EP_RESID) out[v] = r[v] - rp;
  else out[v] = ea + omega * dinv[v] * (r[v] - rp);
}

}  // namespace hc

namespace hc {

// ---------------------------------------------------------------------------------
// z-marching variant: each thread owns one (x, y) column and walks `zc` planes,
// keeping the z-1 / z / z+1 values and labels in registers and prefetching plane
// z+2 one iteration ahead, so every thread has DRAM loads in flight while it
// computes (the one-voxel-per-thread kernel above is latency bound: its unique
// DRAM bytes per thread are too few to cover HBM latency).  x/y neighbours come
// from L1/L2.  Same modes, epilogues and results as k_fine_op.
template <int MODE, int EPI>
__global__ void __launch_bounds__(VX * VY)
k_fine_z(DevParams P, FineArgs F, const double2* __restrict__ V, const double* __restrict__ e,
         const double* __restrict__ r, const double* __restrict__ dinv, double omega,
         double inv_dt, int flags, double2* __restrict__ out2, double* __restrict__ out, int zc) {
  __shared__ double sP[36], sC[36], sM[36];
  __shared__ unsigned char sI[36];
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid < 36) {
    sP[tid] = P.gP[tid];
    sC[tid] = P.gC[tid];
    sM[tid] = P.gMig[tid];
    sI[tid] = P.ifc[tid];
  }
  __syncthreads();
  const int x = blockIdx.x * VX + threadIdx.x, y = blockIdx.y * VY + threadIdx.y;
  if (x >= P.nx || y >= P.ny) return;
  const int nxy = (int)P.nxy, nz = P.nz;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
  if (z0 >= z1) return;
  const int base = y * P.nx + x;
  const double tp = P.t_plus;
  constexpr bool FULLM = MODE == SM_FULL;
  const bool one_c_flag = FULLM && (flags & 4);
  // rolling window (m: z-1, c: z, p: z+1), n: prefetched z+2
  uint8_t lm, lc, lp, ln = 0;
  double2 Vm = {0, 0}, Vc = {0, 0}, Vp = {0, 0}, Vn = {0, 0};
  double em = 0, ec = 0, ep = 0, en = 0;
  double wm = 0, wc = 0, wp = 0, wn = 0;
  auto load = [&](int zz, uint8_t& l, double2& Vv, double& ev, double& wv) {
    const int idx = zz * nxy + base;
    l = __ldg(F.lab + idx);
    if constexpr (FULLM) {
      Vv = V[idx];
      if (one_c_flag) wv = F.w[idx];
    } else {
      ev = e[idx];
    }
  };
  load(z0, lc, Vc, ec, wc);
  if (z0 > 0) load(z0 - 1, lm, Vm, em, wm);
  else { lm = lc; Vm = Vc; em = ec; wm = wc; }
  if (z0 + 1 < nz) load(z0 + 1, lp, Vp, ep, wp);
  else { lp = lc; Vp = Vc; ep = ec; wp = wc; }
  for (int z = z0; z < z1; ++z) {
    const int v = z * nxy + base;
    if (z + 2 < nz && z + 1 < z1) load(z + 2, ln, Vn, en, wn);
    const uint8_t a = lc;
    const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == GR || a == EL)
                                                           : !(z == nz - 1 && a == CC);
    // x/y neighbours of this plane (aliases of v at the domain edge)
    int nb[4];
    nb[0] = x > 0 ? v - 1 : v;
    nb[1] = x + 1 < P.nx ? v + 1 : v;
    nb[2] = y > 0 ? v - P.nx : v;
    nb[3] = y + 1 < P.ny ? v + P.nx : v;
    uint8_t lb[6];
    double2 Vb[6];
    double eb[6], wb[6];
    if (in_row) {
#pragma unroll
      for (int d = 0; d < 4; ++d) {
        lb[d] = __ldg(F.lab + nb[d]);
        if constexpr (FULLM) {
          Vb[d] = V[nb[d]];
          if (one_c_flag) wb[d] = F.w[nb[d]];
        } else {
          eb[d] = e[nb[d]];
        }
      }
      lb[4] = lm; lb[5] = lp;
      if constexpr (FULLM) {
        Vb[4] = Vm; Vb[5] = Vp; wb[4] = wm; wb[5] = wp;
      } else {
        eb[4] = em; eb[5] = ep;
      }
      const int a6 = a * 6;
      bool any_if = false;
#pragma unroll
      for (int d = 0; d < 6; ++d) any_if |= sI[a6 + lb[d]] != 0;
      double rc = 0.0, rp = 0.0;
      if constexpr (FULLM) {
        const double2 Va = Vc;
        const bool one_c = one_c_flag && a == EL;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const int i = a6 + lb[d];
          const double dp = Va.y - Vb[d].y;
          rp += sP[i] * dp;
          rc += sC[i] * (Va.x - Vb[d].x) + sM[i] * dp;
          if (one_c && sM[i] != 0.0) {
            double dq = wc * Va.x - wb[d] * Vb[d].x;
            rp += dq;
            rc += tp * dq;
          }
        }
        if (any_if) {
          const int rk = __ldg(F.if_rank + v);
          const bool solid = a != EL;
#pragma unroll
          for (int d = 0; d < 6; ++d) {
            const uint8_t b = lb[d];
            if (!sI[a6 + b]) continue;
            const long long f = 6LL * rk + d;
            const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f),
                         cg = __ldg(F.vcoef + 2 * F.nslot + f);
            const bool bv = a == GR || b == GR;
            const double2 vs = solid ? Va : Vb[d], ve = solid ? Vb[d] : Va;
            const double dv = (bv ? ca * vs.x : 0.0) + cb * ve.x + cg * (vs.y - ve.y);
            if (solid) {
              if (bv) rc += dv;
              rp += dv;
            } else {
              rc -= dv;
              rp -= dv;
            }
          }
        }
        if ((flags & 1) && (a == GR || a == EL)) rc += Va.x * inv_dt;
        if ((flags & 2) && a == EL) rc -= tp * rp;
        if (flags & 8) rc = 0.0;
        out2[v] = make_double2(rc, rp);
      } else {
        const double ea = ec;
        if (MODE == SM_PHI) {
#pragma unroll
          for (int d = 0; d < 6; ++d) rp += sP[a6 + lb[d]] * (ea - eb[d]);
        } else if (MODE == SM_CONC) {
#pragma unroll
          for (int d = 0; d < 6; ++d) rp += sC[a6 + lb[d]] * (ea - eb[d]);
          rp += inv_dt * ea;
        }
        if (any_if) {
          const int rk = __ldg(F.if_rank + v);
          const bool solid = a != EL;
#pragma unroll
          for (int d = 0; d < 6; ++d) {
            const uint8_t b = lb[d];
            if (!sI[a6 + b]) continue;
            const long long f = 6LL * rk + d;
            const bool bv = a == GR || b == GR;
            if (MODE == SM_PHI) {
              rp += __ldg(F.vcoef + 2 * F.nslot + f) * (ea - eb[d]);
            } else if (MODE == SM_CP) {
              const double cg = __ldg(F.vcoef + 2 * F.nslot + f);
              if (solid) {
                if (bv) rp += cg * (ea - eb[d]);
              } else {
                rp += (1.0 - tp) * cg * (ea - eb[d]);
              }
            } else {
              const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f);
              if (solid) {
                if (bv) rp += ca * ea + cb * eb[d];
              } else {
                rp -= (1.0 - tp) * ((bv ? ca * eb[d] : 0.0) + cb * ea);
              }
            }
          }
        }
        if (EPI == EP_STORE) out[v] = rp;
        else if (EPI == EP_RESID) out[v] = r[v] - rp;
        else out[v] = ea + omega * dinv[v] * (r[v] - rp);
      }
    } else {
      if constexpr (FULLM) out2[v] = make_double2(0.0, 0.0);
      else out[v] = 0.0;
    }
    // advance the window
    lm = lc; Vm = Vc; em = ec; wm = wc;
    lc = lp; Vc = Vp; ec = ep; wc = wp;
    if (z + 2 < nz) { lp = ln; Vp = Vn; ep = en; wp = wn; }
    // (at the top plane z + 1 == nz - 1 the z+1 neighbour aliases the voxel itself)
  }
}

// launch helper: z-chunk length chosen so the grid has >= 4 CTAs per SM
template <int MODE, int EPI>
inline void fine_launch(const DevParams& P, const FineArgs& F, const double2* V, const double* e,
                        const double* r, const double* dinv, double omega, double inv_dt, int flags,
                        double2* out2, double* out, int n_sm, cudaStream_t s) {
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  const long long want = 4LL * n_sm;
  int zc = (int)std::max<long long>(1, (long long)bx * by * P.nz / want);
  zc = std::min(zc, 32);
  const int bz = (P.nz + zc - 1) / zc;
  k_fine_z<MODE, EPI><<<dim3(bx, by, bz), dim3(VX, VY, 1), 0, s>>>(P, F, V, e, r, dinv, omega,
                                                                  inv_dt, flags, out2, out, zc);
}

}  // namespace hc

namespace hc {

// ---------------------------------------------------------------------------------
// 2.5-D tiled variant (the one the solver uses).  A CTA owns a 32 x 8 column of
// the grid and marches `zc` planes.  Each plane's tile plus its one-voxel x/y halo
// (34 x 10 values and labels) is staged in shared memory, double-buffered: the
// global loads of plane z+1 are issued before plane z is computed and land in the
// other buffer afterwards, so DRAM latency overlaps the arithmetic and x/y
// neighbours never go to L2.  z-1 / z+1 values of the own column stay in registers.
// Halo coordinates are clamped into the domain, which aliases every missing
// neighbour to the voxel itself (zero difference -> no face), exactly like the
// reference's face enumeration.
template <int MODE, int EPI>
__global__ void __launch_bounds__(VX * VY)
k_fine_t(DevParams P, FineArgs F, const double2* __restrict__ V, const double* __restrict__ e,
         const double* __restrict__ r, const double* __restrict__ dinv, double omega,
         double inv_dt, int flags, double2* __restrict__ out2, double* __restrict__ out, int zc) {
  constexpr bool FULLM = MODE == SM_FULL;
  constexpr int TW = VX + 2, TH = VY + 2, TN = TW * TH;  // 34 x 10 = 340
  using VT = typename std::conditional<FULLM, double2, double>::type;
  __shared__ VT sv[2][TN];
  __shared__ double sw[FULLM ? 2 : 1][FULLM ? TN : 1];
  __shared__ uint8_t sl[2][TN];
  __shared__ double sP[36], sC[36], sM[36];
  __shared__ unsigned char sI[36];
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid < 36) {
    sP[tid] = P.gP[tid];
    sC[tid] = P.gC[tid];
    sM[tid] = P.gMig[tid];
    sI[tid] = P.ifc[tid];
  }
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  const int x0 = blockIdx.x * VX, y0 = blockIdx.y * VY;
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool active = x < nx && y < ny;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
  const bool one_c_flag = FULLM && (flags & 4);
  // the (up to) two halo elements this thread stages per plane
  int hoff[2];
  bool hval[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * VX * VY;
    hval[k] = i < TN;
    const int hy = i / TW, hx = i - hy * TW;
    const int gx = min(max(x0 + hx - 1, 0), nx - 1), gy = min(max(y0 + hy - 1, 0), ny - 1);
    hoff[k] = gy * nx + gx;
  }
  VT pv[2];
  double pw[2] = {0.0, 0.0};
  uint8_t pl[2];
  auto fetch = [&](int zz) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hval[k]) {
        const int idx = zz * nxy + hoff[k];
        pl[k] = __ldg(F.lab + idx);
        if constexpr (FULLM) {
          pv[k] = V[idx];
          if (one_c_flag) pw[k] = F.w[idx];
        } else {
          pv[k] = e[idx];
        }
      }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hval[k]) {
        const int i = tid + k * VX * VY;
        sl[buf][i] = pl[k];
        sv[buf][i] = pv[k];
        if constexpr (FULLM) sw[buf][i] = pw[k];
      }
  };
  const int cidx = (threadIdx.y + 1) * TW + threadIdx.x + 1;  // own voxel in the tile
  const int col = active ? y * nx + x : 0;
  // own column window: z-1 (m) and z+1 (p)
  VT vm{}, vp{};
  double wm = 0.0, wp = 0.0;
  uint8_t lm = 0, lp = 0;
  if (z0 < z1) {
    fetch(z0);
    stash(0);
    const int zm = z0 > 0 ? z0 - 1 : z0;
    if (active) {
      const int idx = zm * nxy + col;
      lm = __ldg(F.lab + idx);
      if constexpr (FULLM) {
        vm = V[idx];
        if (one_c_flag) wm = F.w[idx];
      } else {
        vm = e[idx];
      }
    }
  }
  const double tp = P.t_plus;
  for (int z = z0; z < z1; ++z) {
    const int buf = (z - z0) & 1;
    const bool has_next = z + 1 < z1;
    if (has_next) fetch(z + 1);
    const int zp = z + 1 < nz ? z + 1 : z;
    double rv = 0.0, dv_ = 0.0;
    int rkv = -1;
    if (active) {
      rkv = __ldg(F.if_rank + z * nxy + col);   // prefetched: interface rows need it
      const int idx = zp * nxy + col;
      lp = __ldg(F.lab + idx);
      if constexpr (FULLM) {
        vp = V[idx];
        if (one_c_flag) wp = F.w[idx];
      } else {
        vp = e[idx];
        if (EPI != EP_STORE) rv = r[z * nxy + col];
        if (EPI == EP_SMOOTH) dv_ = dinv[z * nxy + col];
      }
    }
    __syncthreads();  // plane z staged (and the table loads on the first pass)
    if (active) {
      const int v = z * nxy + col;
      const uint8_t a = sl[buf][cidx];
      const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == GR || a == EL)
                                                             : !(z == nz - 1 && a == CC);
      if (!in_row) {
        if constexpr (FULLM) out2[v] = make_double2(0.0, 0.0);
        else out[v] = 0.0;
      } else {
        const int ti[4] = {cidx - 1, cidx + 1, cidx - TW, cidx + TW};
        uint8_t lb[6];
        VT vb[6];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          lb[d] = sl[buf][ti[d]];
          vb[d] = sv[buf][ti[d]];
        }
        lb[4] = lm; lb[5] = lp;
        vb[4] = vm; vb[5] = vp;
        const VT va = sv[buf][cidx];
        const int a6 = a * 6;
        bool any_if = false;
#pragma unroll
        for (int d = 0; d < 6; ++d) any_if |= sI[a6 + lb[d]] != 0;
        double rc = 0.0, rp = 0.0;
        if constexpr (FULLM) {
          const bool one_c = one_c_flag && a == EL;
          double wa = 0.0, wb[6];
          if (one_c) {
            wa = sw[buf][cidx];
#pragma unroll
            for (int d = 0; d < 4; ++d) wb[d] = sw[buf][ti[d]];
            wb[4] = wm; wb[5] = wp;
          }
#pragma unroll
          for (int d = 0; d < 6; ++d) {
            const int i = a6 + lb[d];
            const double dp = va.y - vb[d].y;
            rp += sP[i] * dp;
            rc += sC[i] * (va.x - vb[d].x) + sM[i] * dp;
            if (one_c && sM[i] != 0.0) {
              double dq = wa * va.x - wb[d] * vb[d].x;
              rp += dq;
              rc += tp * dq;
            }
          }
          if (any_if) {
            const int rk = rkv;
            const bool solid = a != EL;
#pragma unroll
            for (int d = 0; d < 6; ++d) {
              const uint8_t b = lb[d];
              if (!sI[a6 + b]) continue;
              const long long f = 6LL * rk + d;
              const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f),
                           cg = __ldg(F.vcoef + 2 * F.nslot + f);
              const bool bv = a == GR || b == GR;
              const double2 vs = solid ? va : vb[d], ve = solid ? vb[d] : va;
              const double dv = (bv ? ca * vs.x : 0.0) + cb * ve.x + cg * (vs.y - ve.y);
              if (solid) {
                if (bv) rc += dv;
                rp += dv;
              } else {
                rc -= dv;
                rp -= dv;
              }
            }
          }
          if ((flags & 1) && (a == GR || a == EL)) rc += va.x * inv_dt;
          if ((flags & 2) && a == EL) rc -= tp * rp;
          if (flags & 8) rc = 0.0;
          out2[v] = make_double2(rc, rp);
        } else {
          const double ea = va;
          if (MODE == SM_PHI) {
#pragma unroll
            for (int d = 0; d < 6; ++d) rp += sP[a6 + lb[d]] * (ea - vb[d]);
          } else if (MODE == SM_CONC) {
#pragma unroll
            for (int d = 0; d < 6; ++d) rp += sC[a6 + lb[d]] * (ea - vb[d]);
            rp += inv_dt * ea;
          }
          if (any_if) {
            const int rk = rkv;
            const bool solid = a != EL;
#pragma unroll
            for (int d = 0; d < 6; ++d) {
              const uint8_t b = lb[d];
              if (!sI[a6 + b]) continue;
              const long long f = 6LL * rk + d;
              const bool bv = a == GR || b == GR;
              if (MODE == SM_PHI) {
                rp += __ldg(F.vcoef + 2 * F.nslot + f) * (ea - vb[d]);
              } else if (MODE == SM_CP) {
                const double cg = __ldg(F.vcoef + 2 * F.nslot + f);
                if (solid) {
                  if (bv) rp += cg * (ea - vb[d]);
                } else {
                  rp += (1.0 - tp) * cg * (ea - vb[d]);
                }
              } else {
                const double ca = __ldg(F.vcoef + f), cb = __ldg(F.vcoef + F.nslot + f);
                if (solid) {
                  if (bv) rp += ca * ea + cb * vb[d];
                } else {
                  rp -= (1.0 - tp) * ((bv ? ca * vb[d] : 0.0) + cb * ea);
                }
              }
            }
          }
          if (EPI == EP_STORE) out[v] = rp;
          else if (EPI == EP_RESID) out[v] = rv - rp;
          else out[v] = ea + omega * dv_ * (rv - rp);
        }
      }
      // slide the own-column window
      lm = sl[buf][cidx];
      vm = sv[buf][cidx];
      if constexpr (FULLM) wm = sw[buf][cidx];
    }
    if (has_next) stash(buf ^ 1);  // nobody reads buf ^ 1 after the barrier above
  }
}

template <int MODE, int EPI>
inline void fine_launch_t(const DevParams& P, const FineArgs& F, const double2* V, const double* e,
                          const double* r, const double* dinv, double omega, double inv_dt,
                          int flags, double2* out2, double* out, int n_sm, cudaStream_t s) {
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  const long long want = 4LL * n_sm;
  int zc = (int)std::max<long long>(1, (long long)bx * by * P.nz / want);
  zc = std::min(zc, 64);
  const int bz = (P.nz + zc - 1) / zc;
  k_fine_t<MODE, EPI><<<dim3(bx, by, bz), dim3(VX, VY, 1), 0, s>>>(P, F, V, e, r, dinv, omega,
                                                                  inv_dt, flags, out2, out, zc);
}

}  // namespace hc

namespace hc {

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// ---------------------------------------------------------------------------------
// Pipelined 2.5-D stencil (the solver's kernel).  Same tiling as k_fine_t, but the
// plane tiles (values, 32-bit labels, gX/c) are staged with cp.async into a
// 4-deep shared-memory ring: while plane z is computed, planes z+1..z+3 are in
// flight, so every SM keeps several planes of HBM traffic outstanding without
// spending registers on it.  z-1 of the own column is kept in registers, z+1 is
// read from the ring.  The z loop is unrolled by the ring depth so every ring slot
// is a compile-time offset (no per-plane slot arithmetic), and interface faces are
// handled in a second pass only by voxels that own interface slots (the per-voxel
// coefficient rows are zero on non-interface faces).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async4a(unsigned sa, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8a(unsigned sa, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16a(unsigned sa, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
template <int K>
using SlotC = std::integral_constant<int, K>;

template <int MODE, int EPI>
__global__ void __launch_bounds__(VX * VY)
k_fine_p(DevParams P, FineArgs F, const int32_t* __restrict__ lab4, const double2* __restrict__ V,
         const double* __restrict__ e, const double* __restrict__ r, const double* __restrict__ dinv,
         double omega, double inv_dt, int flags, double2* __restrict__ out2, double* __restrict__ out,
         int zc) {
  constexpr bool FULLM = MODE == SM_FULL;
  constexpr bool X0 = EPI == EP_SMOOTH0;   // input e0 = w D^-1 r materialised from staged r, dinv
  constexpr int S = 4;
  constexpr int TW = VX + 2, TH = VY + 2, TN = TW * TH;
  constexpr int VB = FULLM ? 16 : 8;       // bytes per staged value
  using VT = typename std::conditional<FULLM, double2, double>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  VT* sv = reinterpret_cast<VT*>(smem_raw);                       // [S][TN]
  double* sw = reinterpret_cast<double*>(sv + S * TN);             // [S][TN] (FULL only)
  double* sd = sw + (FULLM ? S * TN : 0);                          // [S][TN] dinv (X0 only)
  int* sl = reinterpret_cast<int*>(sd + (X0 ? S * TN : 0));        // [S][TN]
  __shared__ double sP[36], sC[36], sM[36];
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid < 36) {
    sP[tid] = P.gP[tid];
    sC[tid] = P.gC[tid];
    sM[tid] = P.gMig[tid];
  }
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  const int x0 = blockIdx.x * VX, y0 = blockIdx.y * VY;
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool active = x < nx && y < ny;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
  const int zlast = min(z1, nz - 1);  // last plane that must be staged
  const bool one_c_flag = FULLM && (flags & 4);
  // this thread's (up to two) halo elements: global column offset + shared address
  int hoff[2];
  bool hval[2];
  unsigned hsa_l[2], hsa_v[2], hsa_w[2], hsa_d[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * VX * VY;
    hval[k] = i < TN;
    const int hy = i / TW, hx = i - hy * TW;
    const int gx = min(max(x0 + hx - 1, 0), nx - 1), gy = min(max(y0 + hy - 1, 0), ny - 1);
    hoff[k] = gy * nx + gx;
    hsa_l[k] = smem_addr(sl + i);
    hsa_v[k] = smem_addr(sv + i);
    hsa_w[k] = smem_addr(sw + i);
    hsa_d[k] = smem_addr(sd + i);
  }
  const int col = active ? y * nx + x : 0;
  auto issue = [&](int zz, auto slotc) {
    constexpr int buf = decltype(slotc)::value;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hval[k]) {
        const long long idx = (long long)zz * nxy + hoff[k];
        cp_async4a(hsa_l[k] + buf * TN * 4, lab4 + idx);
        if constexpr (FULLM) {
          cp_async16a(hsa_v[k] + buf * TN * VB, V + idx);
          if (one_c_flag) cp_async8a(hsa_w[k] + buf * TN * 8, F.w + idx);
        } else if constexpr (X0) {
          cp_async8a(hsa_v[k] + buf * TN * 8, r + idx);
          cp_async8a(hsa_d[k] + buf * TN * 8, dinv + idx);
        } else {
          cp_async8a(hsa_v[k] + buf * TN * 8, e + idx);
        }
      }
  };
  // staged value -> stencil input (e, or e0 = w dinv r for the zero-guess sweep)
  auto val = [&](int slot) -> VT {
    if constexpr (X0) return omega * sd[slot] * sv[slot];
    else return sv[slot];
  };
  if (z0 <= zlast) issue(z0, SlotC<0>{});
  cp_commit();
  if (z0 + 1 <= zlast) issue(z0 + 1, SlotC<1>{});
  cp_commit();
  if (z0 + 2 <= zlast) issue(z0 + 2, SlotC<2>{});
  cp_commit();
  const int cidx = (threadIdx.y + 1) * TW + threadIdx.x + 1;
  VT vm{};
  double wm = 0.0;
  int lm = 0;
  if (active) {
    const int zm = z0 > 0 ? z0 - 1 : z0;
    const long long idx = (long long)zm * nxy + col;
    lm = lab4[idx] & 7;
    if constexpr (FULLM) {
      vm = V[idx];
      if (one_c_flag) wm = F.w[idx];
    } else if constexpr (X0) {
      vm = omega * dinv[idx] * r[idx];
    } else {
      vm = e[idx];
    }
  }
  const double tp = P.t_plus;
  const long long nslot = F.nslot;
  auto step = [&](int z, auto slotc) {
    constexpr int buf = decltype(slotc)::value;
    constexpr int bufp = (buf + 1) % S;
    const int v = z * nxy + col;
    double rv = 0.0, dv_ = 0.0;
    if (active) {
      if constexpr (!FULLM) {
        if (EPI != EP_STORE) rv = r[v];
        if (EPI == EP_SMOOTH || EPI == EP_SMOOTH0) dv_ = dinv[v];
      }
    }
    cp_wait1();        // planes z and z+1 have landed (only z+2's group may be pending)
    __syncthreads();
    if (z + 3 <= zlast) issue(z + 3, SlotC<(buf + 3) % S>{});  // reuses plane z-1's slot
    cp_commit();
    if (!active) return;
    const int aw = sl[buf * TN + cidx];   // phase | (interface rank + 1) << 3
    const int a = aw & 7;
    const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == GR || a == EL)
                                                           : !(z == nz - 1 && a == CC);
    const bool top = z + 1 >= nz;
    const VT va = val(buf * TN + cidx);
    double wa = 0.0;
    if constexpr (FULLM) wa = one_c_flag ? sw[buf * TN + cidx] : 0.0;
    if (!in_row) {
      if constexpr (FULLM) out2[v] = make_double2(0.0, 0.0);
      else out[v] = 0.0;
    } else {
      const int rk = (aw >> 3) - 1;
      const int a6 = a * 6;
      const bool solid = a != EL;
      double rc = 0.0, rp = 0.0;
      bool one_c = false;
      if constexpr (FULLM) one_c = one_c_flag && a == EL;
      int bb[6];
      VT vbv[6];
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        // neighbour d straight from the ring (z-1 from registers, z+1 from the next slot)
        int b;
        VT vb;
        double wb = 0.0;
        if (d < 4) {
          const int t = d == 0 ? cidx - 1 : (d == 1 ? cidx + 1 : (d == 2 ? cidx - TW : cidx + TW));
          b = sl[buf * TN + t] & 7;
          vb = val(buf * TN + t);
          if constexpr (FULLM) if (one_c) wb = sw[buf * TN + t];
        } else if (d == 4) {
          b = lm;
          vb = vm;
          wb = wm;
        } else {
          b = top ? a : (sl[bufp * TN + cidx] & 7);
          vb = top ? va : val(bufp * TN + cidx);
          if constexpr (FULLM) if (one_c) wb = top ? wa : sw[bufp * TN + cidx];
        }
        bb[d] = b;
        vbv[d] = vb;
        const int i = a6 + b;
        if constexpr (FULLM) {
          const double dp = va.y - vb.y;
          rp += sP[i] * dp;
          rc += sC[i] * (va.x - vb.x) + sM[i] * dp;
          if (one_c && sM[i] != 0.0) {
            const double dq = wa * va.x - wb * vb.x;
            rp += dq;
            rc += tp * dq;
          }
        } else if (MODE == SM_PHI) {
          rp += sP[i] * (va - vb);
        } else if (MODE == SM_CONC) {
          rp += sC[i] * (va - vb);
        }
      }
      if (rk >= 0) {
        // interface kinetics: this voxel's six coefficient slots (zero off-interface)
        const long long f = 6LL * rk;
        double cg[6], ca[6], cb[6];
        if constexpr (FULLM || MODE == SM_PHI || MODE == SM_CP) {
          const double2* q = reinterpret_cast<const double2*>(F.vcoef + 2 * nslot + f);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double2 t = __ldg(q + k);
            cg[2 * k] = t.x;
            cg[2 * k + 1] = t.y;
          }
        }
        if constexpr (FULLM || MODE == SM_CONC) {
          const double2* qa = reinterpret_cast<const double2*>(F.vcoef + f);
          const double2* qb = reinterpret_cast<const double2*>(F.vcoef + nslot + f);
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const double2 ta = __ldg(qa + k), tb = __ldg(qb + k);
            ca[2 * k] = ta.x;
            ca[2 * k + 1] = ta.y;
            cb[2 * k] = tb.x;
            cb[2 * k + 1] = tb.y;
          }
        }
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const bool bv = a == GR || bb[d] == GR;
          const VT vb = vbv[d];
          if constexpr (FULLM) {
            const double2 vs = solid ? va : vb, ve = solid ? vb : va;
            const double dv = (bv ? ca[d] * vs.x : 0.0) + cb[d] * ve.x + cg[d] * (vs.y - ve.y);
            if (solid) {
              if (bv) rc += dv;
              rp += dv;
            } else {
              rc -= dv;
              rp -= dv;
            }
          } else if (MODE == SM_PHI) {
            rp += cg[d] * (va - vb);
          } else if (MODE == SM_CP) {
            if (solid) {
              if (bv) rp += cg[d] * (va - vb);
            } else {
              rp += (1.0 - tp) * cg[d] * (va - vb);
            }
          } else {
            if (solid) {
              if (bv) rp += ca[d] * va + cb[d] * vb;
            } else {
              rp -= (1.0 - tp) * ((bv ? ca[d] * vb : 0.0) + cb[d] * va);
            }
          }
        }
      }
      if constexpr (FULLM) {
        if ((flags & 1) && (a == GR || a == EL)) rc += va.x * inv_dt;
        if ((flags & 2) && a == EL) rc -= tp * rp;
        if (flags & 8) rc = 0.0;
        out2[v] = make_double2(rc, rp);
      } else {
        if (MODE == SM_CONC) rp += inv_dt * va;
        if (EPI == EP_STORE) out[v] = rp;
        else if (EPI == EP_RESID) out[v] = rv - rp;
        else out[v] = va + omega * dv_ * (rv - rp);   // SMOOTH and SMOOTH0
      }
    }
    lm = a;
    vm = va;
    if constexpr (FULLM) wm = wa;
  };
  for (int zb = z0; zb < z1; zb += S) {
    step(zb, SlotC<0>{});
    if (zb + 1 < z1) step(zb + 1, SlotC<1>{});
    if (zb + 2 < z1) step(zb + 2, SlotC<2>{});
    if (zb + 3 < z1) step(zb + 3, SlotC<3>{});
  }
  cp_wait1();
}

// z-chunking for a single wave: as many CTAs as can be resident at once (occupancy
// query, cached per instantiation), each marching ceil(nz / bz) planes — no partial
// last wave, longest possible pipelines.
inline int ctas_per_sm_target() {
  static int t = -1;
  if (t < 0) {
    const char* e = getenv("HC_ZC_TARGET");
    t = e ? atoi(e) : 12;
  }
  return t;
}

// grid z-extent: about `target` CTAs per SM in total (HC_ZC_TARGET; 0 = exactly one
// resident wave from the occupancy query), at least two planes per CTA
inline int pick_bz(int bx, int by, int nz, int per_sm, int n_sm) {
  const int target = ctas_per_sm_target();
  const long long want = (long long)(target > 0 ? target : per_sm) * n_sm;
  int bz = (int)std::max<long long>(1, want / std::max(1, bx * by));
  bz = std::min(bz, std::max(1, nz / 2));
  const int zc = (nz + bz - 1) / bz;
  return (nz + zc - 1) / zc;
}

template <int MODE, int EPI>
inline void fine_launch_p(const DevParams& P, const FineArgs& F, const int32_t* lab4,
                          const double2* V, const double* e, const double* r, const double* dinv,
                          double omega, double inv_dt, int flags, double2* out2, double* out,
                          int n_sm, cudaStream_t s) {
  constexpr bool FULLM = MODE == SM_FULL;
  constexpr int TN = (VX + 2) * (VY + 2);
  const size_t smem = 4 * TN * ((FULLM ? 16 : 8) + (FULLM ? 8 : 0) + (EPI == EP_SMOOTH0 ? 8 : 0) + 4);
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_fine_p<MODE, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_fine_p<MODE, EPI>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fine_p<MODE, EPI>, VX * VY, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  const int bz = pick_bz(bx, by, P.nz, per_sm, n_sm);
  const int zc = (P.nz + bz - 1) / bz;
  k_fine_p<MODE, EPI><<<dim3(bx, by, bz), dim3(VX, VY, 1), smem, s>>>(
      P, F, lab4, V, e, r, dinv, omega, inv_dt, flags, out2, out, zc);
}

}  // namespace hc

namespace hc {

// ---------------------------------------------------------------------------------
// Operator value (residual) stencil with the same cp.async ring: linear two-point
// fluxes, grounded closures, chemical-potential faces (log c, operator.py:322-327),
// boundary drive and implicit-Euler time term.  Interface currents are added by
// k_residual_iface over the compacted face list.
static __global__ void __launch_bounds__(VX * VY)
k_res_p(DevParams P, const int32_t* __restrict__ lab4, const double2* __restrict__ X, double mu,
        int parts, const double* __restrict__ cprev, double inv_dt, double2* __restrict__ out,
        int zc) {
  constexpr int S = 4;
  constexpr int TW = VX + 2, TH = VY + 2, TN = TW * TH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sv = reinterpret_cast<double2*>(smem_raw);
  int* sl = reinterpret_cast<int*>(sv + S * TN);
  __shared__ double sP[36], sC[36], sM[36];
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid < 36) {
    sP[tid] = P.gP[tid];
    sC[tid] = P.gC[tid];
    sM[tid] = P.gMig[tid];
  }
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  const int x0 = blockIdx.x * VX, y0 = blockIdx.y * VY;
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool active = x < nx && y < ny;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
  const int zlast = min(z1, nz - 1);
  int hoff[2];
  bool hval[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = tid + k * VX * VY;
    hval[k] = i < TN;
    const int hy = i / TW, hx = i - hy * TW;
    const int gx = min(max(x0 + hx - 1, 0), nx - 1), gy = min(max(y0 + hy - 1, 0), ny - 1);
    hoff[k] = gy * nx + gx;
  }
  auto issue = [&](int zz, int buf) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (hval[k]) {
        const int i = tid + k * VX * VY;
        const long long idx = (long long)zz * nxy + hoff[k];
        cp_async4(sl + buf * TN + i, lab4 + idx);
        cp_async16(sv + buf * TN + i, X + idx);
      }
  };
  for (int j = 0; j < 3; ++j) {
    if (z0 + j <= zlast) issue(z0 + j, j);
    cp_commit();
  }
  const int cidx = (threadIdx.y + 1) * TW + threadIdx.x + 1;
  const int col = active ? y * nx + x : 0;
  double2 vm{};
  int lm = 0;
  if (active) {
    const int zm = z0 > 0 ? z0 - 1 : z0;
    const long long idx = (long long)zm * nxy + col;
    lm = lab4[idx] & 7;
    vm = X[idx];
  }
  const bool lin = parts & PART_LIN, c1 = parts & PART_1C;
  const double tp = P.t_plus;
  for (int z = z0; z < z1; ++z) {
    const int j = z - z0, buf = j % S, bufp = (j + 1) % S;
    const int v = z * nxy + col;
    double cp = 0.0;
    if (active && (parts & PART_TIME)) cp = cprev[v];
    cp_wait1();
    __syncthreads();
    if (z + 3 <= zlast) issue(z + 3, (j + 3) % S);
    cp_commit();
    if (active) {
      const int a = sl[buf * TN + cidx] & 7;
      const double2 va = sv[buf * TN + cidx];
      const bool grounded_row = z == nz - 1 && a == CC;
      const bool top = z + 1 >= nz;
      if (grounded_row) {
        out[v] = make_double2(0.0, 0.0);
      } else {
        const int a6 = a * 6;
        const bool one_c = c1 && a == EL;
        const double la = one_c ? log(va.x) : 0.0;
        double rc = 0.0, rp = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          int b;
          double2 vb;
          if (d < 4) {
            const int t = d == 0 ? cidx - 1 : (d == 1 ? cidx + 1 : (d == 2 ? cidx - TW : cidx + TW));
            b = sl[buf * TN + t] & 7;
            vb = sv[buf * TN + t];
          } else if (d == 4) {
            b = lm;
            vb = vm;
          } else {
            b = top ? a : (sl[bufp * TN + cidx] & 7);
            vb = top ? va : sv[bufp * TN + cidx];
          }
          const int i = a6 + b;
          if (lin) {
            const double dp = va.y - vb.y;
            rp += sP[i] * dp;
            rc += sC[i] * (va.x - vb.x) + sM[i] * dp;
          }
          if (one_c && sM[i] != 0.0) {   // electrolyte-electrolyte face
            const double q = P.gX * (la - log(vb.x));
            rp += q;
            rc += tp * q;
          }
        }
        if ((parts & PART_BND) && a == CW && z == 0) rp += mu * P.drive;
        if ((parts & PART_TIME) && (a == GR || a == EL)) rc += (va.x - cp) * inv_dt;
        out[v] = make_double2(rc, rp);
      }
      lm = a;
      vm = va;
    }
  }
  cp_wait1();
}

inline void res_launch_p(const DevParams& P, const int32_t* lab4, const double2* X, double mu,
                         int parts, const double* cprev, double inv_dt, double2* out, int n_sm,
                         cudaStream_t s) {
  constexpr int TN = (VX + 2) * (VY + 2);
  const size_t smem = 4 * TN * (16 + 4);
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncSetAttribute(k_res_p, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_res_p, VX * VY, smem);
    if (per_sm < 1) per_sm = 1;
  }
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  const int bz = pick_bz(bx, by, P.nz, per_sm, n_sm);
  const int zc = (P.nz + bz - 1) / bz;
  k_res_p<<<dim3(bx, by, bz), dim3(VX, VY, 1), smem, s>>>(P, lab4, X, mu, parts, cprev, inv_dt,
                                                          out, zc);
}

}  // namespace hc
