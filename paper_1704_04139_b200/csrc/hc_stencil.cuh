// Fused matrix-free Jacobian stencil on the voxel grid (one pass, no atomics).
//
// One thread per voxel row.  All neighbour labels and values are loaded up front
// (clamped indices, masked) so every thread keeps 13+ independent loads in flight;
// the face coefficients are derived from the phase labels, and the linearized
// interface-face derivatives (Butler-Volmer, counter exchange, stripping) are read
// from the compacted face list through the voxel's interface map (if_rank/if_dir),
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

#include "hc_internal.cuh"

namespace hc {

enum { SM_FULL = 0, SM_PHI = 1, SM_CONC = 2, SM_CP = 3 };
enum { EP_STORE = 0, EP_SMOOTH = 1, EP_RESID = 2 };

struct FineArgs {
  const uint8_t* lab;
  const int32_t* if_rank;
  const int32_t* if_dir;
  const double* coef;     // 3 x n_if linearized interface derivatives
  long long n_if;
  const double* w;        // gX / c per electrolyte voxel (FULL with flag 4)
};

template <int MODE, int EPI>
__global__ void __launch_bounds__(256)
k_fine_op(DevParams P, FineArgs F, const double2* __restrict__ V, const double* __restrict__ e,
          const double* __restrict__ r, const double* __restrict__ dinv, double omega,
          double inv_dt, int flags, double2* __restrict__ out2, double* __restrict__ out) {
  const long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  const int x = (int)(v % P.nx);
  const long long t = v / P.nx;
  const int y = (int)(t % P.ny), z = (int)(t / P.ny);
  const uint8_t a = __ldg(F.lab + v);
  const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == GR || a == EL)
                                                         : !(z == P.nz - 1 && a == CC);
  if (!in_row) {
    if (MODE == SM_FULL) out2[v] = make_double2(0.0, 0.0);
    else out[v] = 0.0;
    return;
  }
  long long nb[6];
  bool ok[6];
  ok[0] = x > 0;          nb[0] = ok[0] ? v - 1 : v;
  ok[1] = x + 1 < P.nx;   nb[1] = ok[1] ? v + 1 : v;
  ok[2] = y > 0;          nb[2] = ok[2] ? v - P.nx : v;
  ok[3] = y + 1 < P.ny;   nb[3] = ok[3] ? v + P.nx : v;
  ok[4] = z > 0;          nb[4] = ok[4] ? v - P.nxy : v;
  ok[5] = z + 1 < P.nz;   nb[5] = ok[5] ? v + P.nxy : v;
  uint8_t lb[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) lb[d] = __ldg(F.lab + nb[d]);
  double2 Va, Vb[6];
  double ea = 0.0, eb[6];
  if (MODE == SM_FULL) {
    Va = V[v];
#pragma unroll
    for (int d = 0; d < 6; ++d) Vb[d] = V[nb[d]];
  } else {
    ea = e[v];
#pragma unroll
    for (int d = 0; d < 6; ++d) eb[d] = e[nb[d]];
  }
  const bool one_c = MODE == SM_FULL && (flags & 4) && a == EL;
  double wa = 0.0, wb[6];
  if (one_c) {
    wa = F.w[v];
#pragma unroll
    for (int d = 0; d < 6; ++d) wb[d] = F.w[nb[d]];
  }
  double rc = 0.0, rp = 0.0;  // FULL rows; PHI/CONC accumulate into rp
  const double gM = P.t_plus * P.kappa * P.gF2;
  const double tp = P.t_plus;
  int rk = -2;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    if (!ok[d]) continue;
    const uint8_t b = lb[d];
    const uint8_t k = kind_of(a, b);
    const int zb = d == 4 ? z - 1 : (d == 5 ? z + 1 : z);
    const bool gb = zb == P.nz - 1 && b == CC;
    if (gb) {  // grounded neighbour: conduction closure on the phi row only
      if (MODE != SM_CONC && MODE != SM_CP && (k == K_CONT || k == K_CONTACT)) {
        double g = 2.0 * P.sig[a] * P.sig[b] / (P.sig[a] + P.sig[b]) * P.gF2;
        if (MODE == SM_FULL) rp += g * Va.y; else rp += g * ea;
      }
      continue;
    }
    if (MODE == SM_CP && k != K_BV && k != K_CE && k != K_STRIP) continue;
    if (k == K_CONT) {
      if (MODE == SM_FULL) {
        if (a == GR) {
          rc += P.d_gr * P.inv_h2 * (Va.x - Vb[d].x);
          rp += P.sigma_gr * P.gF2 * (Va.y - Vb[d].y);
        } else if (a == EL) {
          rc += P.d_el * P.inv_h2 * (Va.x - Vb[d].x) + gM * (Va.y - Vb[d].y);
          rp += P.kappa * P.gF2 * (Va.y - Vb[d].y);
          if (one_c) {
            double dq = wa * Va.x - wb[d] * Vb[d].x;
            rp += dq;
            rc += tp * dq;
          }
        } else {
          rp += P.sig[a] * P.gF2 * (Va.y - Vb[d].y);
        }
      } else if (MODE == SM_PHI) {
        double g = (a == GR ? P.sigma_gr : (a == EL ? P.kappa : P.sig[a])) * P.gF2;
        rp += g * (ea - eb[d]);
      } else {
        double g = (a == GR ? P.d_gr : P.d_el) * P.inv_h2;
        rp += g * (ea - eb[d]);
      }
    } else if (k == K_CONTACT) {
      if (MODE != SM_CONC) {
        double g = 2.0 * P.sig[a] * P.sig[b] / (P.sig[a] + P.sig[b]) * P.gF2;
        if (MODE == SM_FULL) rp += g * (Va.y - Vb[d].y); else rp += g * (ea - eb[d]);
      }
    } else if (k == K_BV || k == K_CE || k == K_STRIP) {
      if (rk == -2) rk = __ldg(F.if_rank + v);
      const int f = __ldg(F.if_dir + 6LL * rk + d);
      const double ca = __ldg(F.coef + f), cb = __ldg(F.coef + F.n_if + f),
                   cg = __ldg(F.coef + 2 * F.n_if + f);
      const bool solid = a != EL;
      if (MODE == SM_FULL) {
        // dv = ca c_s + cb c_e + cg (phi_s - phi_e)  (ca = 0 unless BV)
        const double2 vs = solid ? Va : Vb[d], ve = solid ? Vb[d] : Va;
        double dv = (k == K_BV ? ca * vs.x : 0.0) + cb * ve.x + cg * (vs.y - ve.y);
        if (solid) {
          if (k == K_BV) rc += dv;
          rp += dv;
        } else {  // the row transform T is applied once below (rc -= t+ rp)
          rc -= dv;
          rp -= dv;
        }
      } else if (MODE == SM_PHI) {
        rp += cg * (ea - eb[d]);
      } else if (MODE == SM_CP) {
        if (solid) {
          if (k == K_BV) rp += cg * (ea - eb[d]);
        } else {
          rp += (1.0 - tp) * cg * (ea - eb[d]);
        }
      } else {
        if (solid) {
          if (k == K_BV) rp += ca * ea + cb * eb[d];
        } else {
          rp -= (1.0 - tp) * ((k == K_BV ? ca * eb[d] : 0.0) + cb * ea);
        }
      }
    }
  }
  if (MODE == SM_FULL) {
    const bool has_c = a == GR || a == EL;
    if ((flags & 1) && has_c) rc += Va.x * inv_dt;
    if ((flags & 2) && a == EL) rc -= tp * rp;
    if (flags & 8) rc = 0.0;
    out2[v] = make_double2(rc, rp);
  } else {
    if (MODE == SM_CONC) rp += inv_dt * ea;
    // SM_CP with EP_RESID: out = r - (T J)_cp e (the c-block right-hand side)
    if (EPI == EP_STORE) out[v] = rp;
    else if (EPI == EP_RESID) out[v] = r[v] - rp;
    else out[v] = ea + omega * dinv[v] * (r[v] - rp);
  }
}

}  // namespace hc
