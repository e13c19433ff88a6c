// Fused matrix-free Jacobian stencil on the voxel grid (one pass, no atomics).
//
// The face coefficients are derived from the phase labels, and the linearized
// interface-face derivatives (Butler-Volmer, counter exchange, stripping) are read
// per (interface voxel, direction) through the voxel's interface rank, oriented
// from the row's side, so interface faces need no separate kernel and no atomics.
// This file holds the cp.async ring variant (any grid); hc_tma.cuh holds the TMA
// variant the solver uses when the x pitch allows tensor-map tiles.
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
enum { EP_STORE = 0, EP_SMOOTH = 1, EP_RESID = 2, EP_SMOOTH0 = 3, EP_RESID0 = 4 };
// SMOOTH0: first sweep from e0 = w D^-1 r;  RESID0: r - A e0 with e0 = w D^-1 r, and e0 itself
// written to the double* passed as out2 (the zero-guess smoothing step and the residual in one pass)

struct FineArgs {
  const uint8_t* lab;
  const int32_t* if_rank;
  const double* vcoef;    // interface derivatives per (interface voxel, direction): [3][nslot]
  long long nslot;        // 6 * number of interface voxels
  const double* w;        // gX / c per electrolyte voxel (FULL with flag 4)
  const double* cslot;    // TMA stencil: compact row-oriented (alpha, beta, gamma) per interface face slot
  const int2* elz;        // TMA stencil: per 32 x 8 tile column, z range holding electrolyte (lo, hi)
  const double* islot;    // TMA residual: interface current per face slot, oriented from the row
  const int32_t* tp_off;  // TMA stencil: first face slot of every (32 x 8 tile, plane), + total
  // TMA J v only: per-CTA partial dot products of the output with dot_a (and, dot_two,
  // with itself) into dot_part[cta] / dot_part[n_cta + cta]; the launcher stores n_cta in
  // *dot_nblk (host).  Lets BiCGStab drop its separate reduction pass after each J v.
  const double2* dot_a = nullptr;
  double* dot_part = nullptr;
  int dot_two = 0;
  int* dot_nblk = nullptr;
  // TMA c-block sweeps (CONC / CP): planes [cz.x, cz.y) hold every c row (electrolyte and
  // graphite voxels); empty (0, 0): sweep the whole grid
  int2 cz = {0, 0};
};

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
  pdl_wait();
  constexpr bool FULLM = MODE == SM_FULL;
  constexpr bool X0 = EPI == EP_SMOOTH0 || EPI == EP_RESID0;   // input e0 = w D^-1 r from staged r, dinv
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
      else out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = 0.0;
    } else {
      const int rk = (aw >> 3) - 1;
      const int a6 = a * 6;
      const bool solid = a != EL;
      double rc = 0.0, rp = 0.0;
      bool one_c = false;
      if constexpr (FULLM) one_c = one_c_flag && a == EL;
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
        // interface kinetics: six row-oriented coefficient triples (zero off-interface),
        // each face adds alpha c_a + beta c_b + gamma (phi_a - phi_b) to the phi row
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
        double si = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const VT vb = vbv[d];
          if constexpr (FULLM) si += ca[d] * va.x + cb[d] * vb.x + cg[d] * (va.y - vb.y);
          else if (MODE == SM_CONC) si += ca[d] * va + cb[d] * vb;
          else si += cg[d] * (va - vb);
        }
        if constexpr (FULLM) {
          rp += si;
          if (a == GR || a == EL) rc += si;
        } else if (MODE == SM_PHI) {
          rp += si;
        } else {
          rp += (solid ? 1.0 : 1.0 - tp) * si;   // (T J) on electrolyte c rows
        }
      }
      if constexpr (FULLM) {
        if ((flags & 1) && (a == GR || a == EL)) rc += va.x * inv_dt;
        if ((flags & 2) && a == EL) rc -= tp * rp;
        if (flags & 8) rc = 0.0;
        out2[v] = make_double2(rc, rp);
      } else {
        if (MODE == SM_CONC) rp += inv_dt * va;
        if (EPI == EP_STORE) out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = rp;
        else if (EPI == EP_RESID || EPI == EP_RESID0) out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = rv - rp;
        else out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = va + omega * dv_ * (rv - rp);   // SMOOTH and SMOOTH0
      }
    }
    if constexpr (EPI == EP_RESID0) reinterpret_cast<double*>(out2)[v] = va;
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
    t = e ? atoi(e) : 6;
  }
  return t;
}
inline int min_planes_per_cta() {
  static int t = -1;
  if (t < 0) {
    const char* e = getenv("HC_ZC_MIN");
    t = std::max(1, e ? atoi(e) : 5);
  }
  return t;
}

// grid z-extent: about `target` CTAs per SM in total (HC_ZC_TARGET; 0 = exactly one
// resident wave from the occupancy query), at least HC_ZC_MIN planes per CTA (every
// CTA pays a pipeline fill and re-reads its first and last neighbour planes)
inline int pick_bz(int bx, int by, int nz, int per_sm, int n_sm) {
  const int target = ctas_per_sm_target();
  const long long want = (long long)(target > 0 ? target : per_sm) * n_sm;
  int bz = (int)std::max<long long>(1, want / std::max(1, bx * by));
  // grids too small to give every SM a CTA at the usual minimum march on 2 planes per CTA
  // instead (tiny cell, 4 tile columns: 48 -> 128 CTAs, 7.10 -> 6.43 ms per step; the medium and
  // batched cells already fill the GPU and measured slower with shorter marches)
  static const bool min_forced = getenv("HC_ZC_MIN") != nullptr;
  int minp = min_planes_per_cta();
  if (!min_forced && (long long)bx * by * (nz / minp) < n_sm) minp = 2;
  bz = std::min(bz, std::max(1, nz / minp));
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
  const size_t smem = 4 * TN * ((FULLM ? 16 : 8) + (FULLM ? 8 : 0) + (EPI == EP_SMOOTH0 || EPI == EP_RESID0 ? 8 : 0) + 4);
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
  launch(k_fine_p<MODE, EPI>, dim3(bx, by, bz), dim3(VX, VY, 1), smem, s, P, F, lab4, V, e, r, dinv, omega,
         inv_dt, flags, out2, out, zc);
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
