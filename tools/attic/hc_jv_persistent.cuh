// Persistent TMA-fed J v stencil (the Krylov operator, SM_FULL).
//
// Same tiles, ring and face word as k_fine_tma (hc_tma.cuh); what differs:
//  * persistent CTAs: the (32 x 8 tile column, plane) units of the grid are split evenly
//    over exactly one resident wave of CTAs; a CTA's range may continue into the next
//    tile column (the ring keeps running across the switch), so there is no partial
//    second wave and one pipeline fill per CTA;
//  * warp-uniform plain paths: a warp none of whose 32 voxels has an interface face, a
//    contact face or a grounded row (one mask test on the face word and a vote) skips the
//    interface and contact code, and runs the conduction sums of its phase class only:
//    all metal -> phi; no electrolyte lane -> (c, phi); else (c, phi, gX/c);
//  * interface faces are walked by set bit of the voxel's interface mask (as many
//    iterations as the busiest lane has faces) instead of six predicated blocks;
//  * the fused dot-product operand is fetched at the top of the plane step;
//  * no face-word tile: a voxel needs only its own face word (the conduction mask replaced
//    the neighbour labels), so each thread reads it straight from global memory one plane
//    ahead — the ring stages shrink and one more stage fits per CTA;
//  * a warp releases a ring stage as soon as it has read its neighbours from it, before
//    the arithmetic and the store: more stages are in flight (the kernel is bound by
//    TMA bytes in flight x latency, not by instruction issue);
//  * face slots past the staged capacity are prefetched into L2 by the producer.
// Differences va - vb are formed before they are summed (as in k_fine_tma): on metal rows
// the face coefficient is ~1e10 times the row's net value, and the sum of differences
// keeps the cancellation exact where 6 va - sum(vb) would not.
#pragma once

#include "hc_tma.cuh"

namespace hc {

#ifndef HC_JV_NOINLINE
#define HC_JV_NOINLINE 0
#endif
#ifndef HC_JV_REM
#define HC_JV_REM 0
#endif
#ifndef HC_JV_PF
#define HC_JV_PF 0
#endif
#ifndef HC_JV_EARLY
#define HC_JV_EARLY 0
#endif
#ifndef HC_JV_SELF
#define HC_JV_SELF 0
#endif
constexpr bool JV_EARLY = HC_JV_EARLY;
#ifndef HC_JV_STAGES
#define HC_JV_STAGES 4
#endif
#ifndef HC_JV_SLOTCAP
#define HC_JV_SLOTCAP 256
#endif
constexpr int JV_S = HC_JV_STAGES;      // ring depth
constexpr int JV_CAP = HC_JV_SLOTCAP;   // interface face slots staged per (tile, plane)
// one ring stage: own face words 32 x 8 int32 | values 34 x 10 double2 | gX/c 36 x 10 double | face slots
struct JvLayout {
  static constexpr int LAB = 0;
  static constexpr int LBYTES = VX * VY * 4;
  static constexpr int VAL = LBYTES;
  static constexpr int VBYTES = T_QN * 16;
  static constexpr int AUX = VAL + ((VBYTES + 127) / 128) * 128;
  static constexpr int SLT = AUX + ((T_DN * 8 + 127) / 128) * 128;
  static constexpr int SLOT = SLT + ((JV_CAP + 2) * 32 + 127) / 128 * 128;
  static constexpr int THREADS = VX * (VY + 1);
};

constexpr unsigned JV_PLAINM = (63u << 3) | (unsigned)FW_CONTACT | (unsigned)FW_GROUND;
constexpr int TPL = PL + 1;   // first metal phase in the TMA label encoding (PL, FOIL, CW, CC)

__device__ __forceinline__ void tma_prefetch3(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

// interface faces of a voxel whose slots were not staged (tile-planes with more than JV_CAP
// slots): the same walk as in the kernel, slots read from global memory
__device__ __noinline__ double jv_faces_global(const double* __restrict__ cs, unsigned mask, double2 va,
                                               double2 vm, double2 v1, const double2* own) {
  double si = 0.0;
  do {
    const int d = __ffs(mask) - 1;
    mask &= mask - 1;
    const int o = (d & 2) ? ((d & 1) ? T_QW : -T_QW) : ((d & 1) ? 1 : -1);
    double2 vbd = d == 4 ? vm : v1;
    if (d < 4) vbd = own[o];
    si += cs[0] * va.x + cs[1] * vbd.x + cs[2] * (va.y - vbd.y);
    cs += 4;
  } while (mask);
  return si;
}

template <bool OC, bool DOT>
__global__ void __launch_bounds__(T_THREADS, HC_TMA_MINB)
k_jv_tma(DevParams P, const __grid_constant__ TmaMaps M, FineArgs F, const int32_t* __restrict__ labt,
         const double2* __restrict__ V, double inv_dt, int flags, double2* __restrict__ out2, int tbx,
         int tby, const int32_t* __restrict__ bounds) {
  using L = JvLayout;
  extern __shared__ __align__(16) unsigned char smem_dyn[];
  unsigned char* ring = smem_dyn + ((128 - ((unsigned)__cvta_generic_to_shared(smem_dyn) & 127)) & 127);
  __shared__ __align__(16) double2 sPC[64];   // (P, C) per (a << 3 | b): contact voxels
  __shared__ __align__(16) double2 sSelf[8];  // (P, C) of a phase's same-phase faces
  __shared__ int tp_start[JV_S];
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  // the mbarriers live behind the ring, so their addresses are the ring base plus a constant
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(ring) + JV_S * L::SLOT;
  const unsigned empty0 = full0 + 8 * JV_S;
  const int tid = threadIdx.y * VX + threadIdx.x;
  // this CTA's share of the (tile column, plane) units, column-major: contiguous ranges of
  // about equal cost (plain metal planes are cheap, interface-rich planes are not)
  const long long u0 = bounds[blockIdx.x], u1 = bounds[blockIdx.x + 1];
  if (tid == T_WARPS * VX) {
#pragma unroll
    for (int k = 0; k < JV_S; ++k) {
      mbar_init(full0 + 8 * k, 1);
      mbar_init(empty0 + 8 * k, T_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 64) {
    const int a = tid >> 3, b = tid & 7;
    const bool ok = a >= 1 && a <= N_PHASES && b >= 1 && b <= N_PHASES;
    const int i = (a - 1) * 6 + (b - 1);
    sPC[tid] = ok ? make_double2(P.gP[i], P.gC[i]) : make_double2(0.0, 0.0);
    if (tid < 8) {
      const bool sk = tid >= 1 && tid <= N_PHASES;
      sSelf[tid] = sk ? make_double2(P.gP[7 * (tid - 1)], P.gC[7 * (tid - 1)]) : make_double2(0.0, 0.0);
    }
  }
  __syncthreads();   // barriers initialised, tables built (the only CTA-wide barrier)
  pdl_wait();

  if (threadIdx.y == T_WARPS) {   // ---------------- producer warp
    const int lane = threadIdx.x;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(ring);
    constexpr unsigned tx_bytes = L::LBYTES + L::VBYTES;
    unsigned round = 0;   // ring rounds completed so far (all segments)
    for (long long u = u0; u < u1;) {
      const int c = (int)(u / nz), za = (int)(u - (long long)c * nz);
      const int zb = (int)min((long long)nz, (long long)za + (u1 - u));
      const int ty = c / tbx, tx = c - ty * tbx;
      const int x0 = tx * VX, y0 = ty * VY;
      int2 elz = make_int2(0, -1);
      if constexpr (OC) elz = F.elz[c];
      const int nst = zb - za + 1;   // planes za .. zb are staged, za .. zb - 1 computed
      // every segment starts at ring slot 0 (compile-time slots in the compute warps): the
      // last round is padded with empty stages (an arrive without data)
      const int npad = (nst + JV_S - 1) / JV_S * JV_S;
      int st_l = 0, cnt_l = 0;
      for (int j = 0; j < npad; ++j) {
        if ((j & 31) == 0) {   // first face slot / slot count of the next 32 tile-planes, lane-parallel
          const int zz = za + j + lane;
          st_l = cnt_l = 0;
          if (j + lane < nst && zz < nz) {
            const long long tpi = ((long long)zz * tby + ty) * tbx + tx;
            st_l = F.tp_off[tpi];
            cnt_l = F.tp_off[tpi + 1] - st_l;
          }
        }
        const int st = __shfl_sync(0xffffffffu, st_l, j & 31), tot = __shfl_sync(0xffffffffu, cnt_l, j & 31);
        const int cnt = min(tot, JV_CAP);
        const unsigned slot = j % JV_S;
        if (lane == 0) {
          if (round) mbar_wait(empty0 + 8 * slot, (round - 1) & 1);
          const unsigned b = full0 + 8 * slot, s = sbase + slot * L::SLOT;
          if (j < nst) {
            const int zz = za + j;
            const bool wtile = OC && zz >= elz.x - 1 && zz <= elz.y + 1;
            tp_start[slot] = st;
            mbar_expect_tx(b, tx_bytes + (wtile ? T_DN * 8 : 0) + 32u * cnt);
            if (HC_JV_PF > 0 && zz + HC_JV_PF < nz) {
              // warm L2 for the plane HC_JV_PF ahead: the ring's own loads then see L2 latency
              const int zp = zz + HC_JV_PF;
              tma_prefetch3(&M.val, 2 * (x0 - T_QOFF), y0 - 1, zp);
              if (OC && zp >= elz.x - 1 && zp <= elz.y + 1) tma_prefetch3(&M.aux, x0 - T_DOFF, y0 - 1, zp);
              tma_prefetch3(&M.lab, x0, y0, zp);
            }
            tma_load3(s + L::LAB, &M.lab, x0, y0, zz, b);
            tma_load3(s + L::VAL, &M.val, 2 * (x0 - T_QOFF), y0 - 1, zz, b);
            if (wtile) tma_load3(s + L::AUX, &M.aux, x0 - T_DOFF, y0 - 1, zz, b);
            if (cnt) bulk_load(s + L::SLT, F.cslot + 4LL * st, 32u * cnt, b);
            if (tot > cnt)   // the few slots past the staged capacity are read from global: warm L2
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(F.cslot + 4LL * (st + cnt)),
                           "r"(32u * (unsigned)(tot - cnt))
                           : "memory");
          } else {
            mbar_arrive(b);
          }
        }
        if (slot == JV_S - 1) ++round;
        __syncwarp();
      }
      u += zb - za;
    }
    return;
  }

  // ---------------------------------------------------- compute warps
  const double tp = P.t_plus;
  const bool f_mass = flags & 1, f_T = flags & 2, f_zc = flags & 8;
  // a warp owns an 8 x 4 patch of the 32 x 8 tile (4 x 2 patches): compact patches cross
  // phase boundaries less often than 32 x 1 rows, so fewer warps leave the plain path
  // (large cell: 28.5 % against 41.5 %); a quarter warp still reads 128 contiguous bytes
  const int px = 8 * (threadIdx.y & 3) + (threadIdx.x & 7), py = 4 * (threadIdx.y >> 2) + (threadIdx.x >> 3);
  // byte offsets of the own voxel inside a slot
  const int aofs = L::AUX + 8 * ((py + 1) * T_DW + px + T_DOFF);
  const int vofs = L::VAL + 16 * ((py + 1) * T_QW + px + T_QOFF);
  const int lofs = L::LAB + 4 * (py * VX + px);
  auto lab_own = [&](const unsigned char* Sx) -> int { return *reinterpret_cast<const int*>(Sx + lofs); };
  auto val_at = [&](const unsigned char* Sx, int o) -> double2 {
    return *reinterpret_cast<const double2*>(Sx + vofs + 16 * o);
  };
  auto phi_at = [&](const unsigned char* Sx, int o) -> double {
    return *reinterpret_cast<const double*>(Sx + vofs + 16 * o + 8);
  };
  auto w_at = [&](const unsigned char* Sx, int o) -> double {
    return *reinterpret_cast<const double*>(Sx + aofs + 8 * o);
  };
  unsigned rnd = 0;   // ring rounds completed so far (all segments)
  double dacc1 = 0.0, dacc2 = 0.0;
  for (long long u = u0; u < u1;) {
    const int c = (int)(u / nz), za = (int)(u - (long long)c * nz);
    const int zb = (int)min((long long)nz, (long long)za + (u1 - u));
    const int ty = c / tbx, tx = c - ty * tbx;
    const int x = tx * VX + px, y = ty * VY + py;
    const bool active = x < nx && y < ny;
    const int col = active ? y * nx + x : 0;
    const int nplane = zb - za;
    const unsigned r0 = rnd;   // ring round at the segment's first stage
    double2 vm = make_double2(0.0, 0.0);   // own column at z - 1
    double wm = 0.0;
    int lm = 0;
    if (active && za > 0) {
      const long long idx = (long long)(za - 1) * nxy + col;
      lm = labt[idx] & 7;
      vm = V[idx];
      if constexpr (OC) wm = F.w[idx];
    }
    mbar_wait(full0, rnd & 1);
    int aw = lab_own(ring);
    double2 va = val_at(ring, 0);
    double wa = 0.0;
    if constexpr (OC) wa = w_at(ring, 0);
    // one plane; K is the ring slot of plane j (a compile-time constant in the unrolled
    // rounds, a register in the segment's last partial round)
    auto step = [&](int j, const int K, unsigned ph1) {
      const int K1 = K + 1 == JV_S ? 0 : K + 1;
      const unsigned char* S0 = ring + K * L::SLOT;
      const unsigned char* S1 = ring + K1 * L::SLOT;
      const int v = (za + j) * nxy + col;
      double2 da = make_double2(0.0, 0.0);
      if constexpr (DOT) {
        if (active) da = F.dot_a[v];
      }
      mbar_wait(full0 + 8 * K1, ph1);
      // own column at z + 1: the z + 1 neighbour now, the own voxel of the next plane
      const int aw1 = lab_own(S1);
      const double2 v1 = val_at(S1, 0);
      double w1 = 0.0;
      if constexpr (OC) w1 = w_at(S1, 0);
      const int a = aw & 7;
      const unsigned sm = ((unsigned)aw >> FW_SELF) & 63u;   // same-phase conduction faces
      // this warp is done with plane j's stage once its neighbours are in registers
      auto release_now = [&]() {
        __syncwarp();
        if (threadIdx.x == 0) mbar_arrive(empty0 + 8 * K);
      };
      auto release = [&]() {
        if constexpr (JV_EARLY) release_now();
      };
      // plain voxel: no interface face, no contact face, not grounded — only same-phase
      // conduction faces (missing or blocked neighbours are simply not in the mask)
      const bool plain = active && !((unsigned)aw & JV_PLAINM);
      double rc = 0.0, rp = 0.0;
      if (__all_sync(0xffffffffu, plain)) {
        const double2 ps = sSelf[a];
#if HC_JV_SELF
        // a face that is not in the mask reads the own value: its difference is exactly zero
        if (__all_sync(0xffffffffu, a >= TPL)) {
          // metals: no c unknown, phi only
          const double p0 = (sm & 1u) ? phi_at(S0, -1) : va.y, p1 = (sm & 2u) ? phi_at(S0, 1) : va.y;
          const double p2 = (sm & 4u) ? phi_at(S0, -T_QW) : va.y, p3 = (sm & 8u) ? phi_at(S0, T_QW) : va.y;
          release();
          const double p4 = (sm & 16u) ? vm.y : va.y, p5 = (sm & 32u) ? v1.y : va.y;
          rp = ps.x * (((va.y - p0) + (va.y - p1)) + ((va.y - p2) + (va.y - p3)) + ((va.y - p4) + (va.y - p5)));
        } else {
          const double2 n0 = (sm & 1u) ? val_at(S0, -1) : va, n1 = (sm & 2u) ? val_at(S0, 1) : va;
          const double2 n2 = (sm & 4u) ? val_at(S0, -T_QW) : va, n3 = (sm & 8u) ? val_at(S0, T_QW) : va;
          const double2 n4 = (sm & 16u) ? vm : va, n5 = (sm & 32u) ? v1 : va;
          const double dp = ((va.y - n0.y) + (va.y - n1.y)) + ((va.y - n2.y) + (va.y - n3.y)) +
                            ((va.y - n4.y) + (va.y - n5.y));
          const double dc = ((va.x - n0.x) + (va.x - n1.x)) + ((va.x - n2.x) + (va.x - n3.x)) +
                            ((va.x - n4.x) + (va.x - n5.x));
          rp = ps.x * dp;
          rc = ps.y * dc;
          if (OC && __any_sync(0xffffffffu, a == TEL)) {
            // gX/c terms of electrolyte rows: sum over faces of (w_a c_a - w_b c_b)
            const double u = wa * va.x;
            const double u0 = (sm & 1u) ? w_at(S0, -1) * n0.x : u, u1 = (sm & 2u) ? w_at(S0, 1) * n1.x : u;
            const double u2 = (sm & 4u) ? w_at(S0, -T_DW) * n2.x : u, u3 = (sm & 8u) ? w_at(S0, T_DW) * n3.x : u;
            release();
            const double u4 = (sm & 16u) ? wm * vm.x : u, u5 = (sm & 32u) ? w1 * v1.x : u;
            const double q = ((u - u0) + (u - u1)) + ((u - u2) + (u - u3)) + ((u - u4) + (u - u5));
            if (a == TEL) rp += q;
          } else {
            release();
          }
          if (a == TEL && !f_T) rc = fma(tp, rp, rc);   // migration + chemical potential: t+ x phi-row terms
          if (f_mass && a <= TGR) rc = fma(va.x, inv_dt, rc);
        }
#else
        auto nbv = [&](int d) -> double2 {
          if (d == 4) return vm;
          if (d == 5) return v1;
          return val_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_QW : T_QW)));
        };
        auto nbp = [&](int d) -> double {
          if (d == 4) return vm.y;
          if (d == 5) return v1.y;
          return phi_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_QW : T_QW)));
        };
        auto nbw = [&](int d) -> double {
          if (d == 4) return wm;
          if (d == 5) return w1;
          return w_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_DW : T_DW)));
        };
        if (__all_sync(0xffffffffu, a >= TPL)) {
          double dp = 0.0;
#pragma unroll
          for (int d = 0; d < 6; ++d)
            if (sm & (1u << d)) dp += va.y - nbp(d);
          release();
          rp = ps.x * dp;
        } else if (!OC || !__any_sync(0xffffffffu, a == TEL)) {
          double dp = 0.0, dc = 0.0;
#pragma unroll
          for (int d = 0; d < 6; ++d)
            if (sm & (1u << d)) {
              const double2 vbd = nbv(d);
              dp += va.y - vbd.y;
              dc += va.x - vbd.x;
            }
          release();
          rp = ps.x * dp;
          rc = ps.y * dc;
          if (a == TEL && !f_T) rc = fma(tp, rp, rc);
          if (f_mass && a <= TGR) rc = fma(va.x, inv_dt, rc);
        } else {
          double dp = 0.0, dc = 0.0, q = 0.0;
#pragma unroll
          for (int d = 0; d < 6; ++d)
            if (sm & (1u << d)) {
              const double2 vbd = nbv(d);
              dp += va.y - vbd.y;
              dc += va.x - vbd.x;
              q = fma(-nbw(d), vbd.x, q);
            }
          release();
          rp = ps.x * dp;
          rc = ps.y * dc;
          if (a == TEL) {
            rp += fma((double)__popc(sm), wa * va.x, q);
            if (!f_T) rc = fma(tp, rp, rc);
          }
          if (f_mass && a <= TGR) rc = fma(va.x, inv_dt, rc);
        }
#endif
        if (f_zc) rc = 0.0;
      } else {
        // neighbour d: 0 x-1, 1 x+1, 2 y-1, 3 y+1, 4 z-1 (registers), 5 z+1 (registers)
        auto nb_val = [&](int d) -> double2 {
          if (d == 4) return vm;
          if (d == 5) return v1;
          return val_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_QW : T_QW)));
        };
        auto nb_w = [&](int d) -> double {
          if (d == 4) return wm;
          if (d == 5) return w1;
          return w_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_DW : T_DW)));
        };
        if (active && !(aw & FW_GROUND)) {
          const bool elrow = a == TEL;
          const bool crow = a == TGR || elrow;
          if (aw & FW_CONTACT) {
            // rare (solid conductors touching another conductor phase): the (P, C) table of
            // the face's phase pair on every face; the in-plane neighbours' phases come from
            // their face words in global memory.  Never an electrolyte row.
            const int a8 = a << 3;
#pragma unroll
            for (int d = 0; d < 6; ++d) {
              int lb;
              if (d == 4) lb = lm;
              else if (d == 5) lb = aw1 & 7;
              else {
                const bool in = d == 0 ? x > 0 : (d == 1 ? x + 1 < nx : (d == 2 ? y > 0 : y + 1 < ny));
                lb = in ? (labt[v + (d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -nx : nx)))] & 7) : 0;
              }
              const double2 pc = sPC[a8 | lb];
              const double2 vbd = nb_val(d);
              rp = fma(pc.x, va.y - vbd.y, rp);
              rc = fma(pc.y, va.x - vbd.x, rc);
            }
          } else {
            const double2 ps = sSelf[a];
            double dp = 0.0, dc = 0.0, q = 0.0;
#pragma unroll
            for (int d = 0; d < 6; ++d)
              if (sm & (1u << d)) {
                const double2 vbd = nb_val(d);
                dp += va.y - vbd.y;
                dc += va.x - vbd.x;
                if constexpr (OC) q = fma(-nb_w(d), vbd.x, q);   // gX/c: electrolyte rows only
              }
            rp = ps.x * dp;
            rc = ps.y * dc;
            if constexpr (OC) {
              q = fma((double)__popc(sm), wa * va.x, q);
              rp += elrow ? q : 0.0;
            }
          }
          // interface kinetics: the voxel's face slots, consecutive in direction order from the
          // tile-plane-local index in its word (staged with the plane; global past capacity);
          // face d adds alpha c_a + beta c_b + gamma (phi_a - phi_b) to the phi row.  Walked by
          // set bit of the interface mask: as many iterations as the busiest lane has faces.
          double si = 0.0;
          unsigned mask = ((unsigned)aw >> 3) & 63u;
          if (mask) {
            const int loc = (int)((unsigned)aw >> FW_SLOT), n = __popc(mask);
            auto faces = [&](const double* cs) {
              do {
                const int d = __ffs(mask) - 1;
                mask &= mask - 1;
                const int o = (d & 2) ? ((d & 1) ? T_QW : -T_QW) : ((d & 1) ? 1 : -1);
                double2 vbd = d == 4 ? vm : v1;
                if (d < 4) vbd = val_at(S0, o);
                const double2 ab = *reinterpret_cast<const double2*>(cs);
                const double g = cs[2];
                si += ab.x * va.x + ab.y * vbd.x + g * (va.y - vbd.y);
                cs += 4;
              } while (mask);
            };
            if (loc + n <= JV_CAP)
              faces(reinterpret_cast<const double*>(S0 + L::SLT) + 4 * loc);
#if HC_JV_NOINLINE
            else   // past the staged capacity (rare): slots from global memory, out of line
              si = jv_faces_global(F.cslot + 4LL * (tp_start[K] + loc), mask, va, vm, v1,
                                   reinterpret_cast<const double2*>(S0 + vofs));
#else
            else faces(F.cslot + 4LL * (tp_start[K] + loc));
#endif
          }
          if (elrow) rc = f_T ? fma(1.0 - tp, si, rc) : fma(tp, rp, rc) + si;   // T: c -= t+ phi
          else if (crow) rc += si;
          rp += si;
          if (f_mass && crow) rc = fma(va.x, inv_dt, rc);
          if (f_zc) rc = 0.0;
        }
        release();
      }
      if constexpr (!JV_EARLY) release_now();
      if (active) {
        out2[v] = make_double2(rc, rp);
        if constexpr (DOT) {
          dacc1 += rc * da.x + rp * da.y;
          dacc2 += rc * rc + rp * rp;
        }
      }
      lm = a;
      vm = va;
      if constexpr (OC) {
        wm = wa;
        wa = w1;
      }
      aw = aw1;
      va = v1;
    };
    // unrolled by the ring depth (slots are compile-time); whole rounds first, so the four
    // steps of a round are straight-line code, then the segment's last partial round
    int jb = 0;
    for (; jb + JV_S <= nplane; jb += JV_S, ++rnd) {
      static_for<JV_S>([&](auto kc) {
        constexpr int K = decltype(kc)::value;
        step(jb + K, K, (K + 1 == JV_S ? rnd + 1 : rnd) & 1);
      });
    }
    // the last partial round (at most JV_S - 1 planes): one not-unrolled copy of the step
#if HC_JV_REM
#pragma unroll 1
    for (int k = 0; jb + k < nplane; ++k) step(jb + k, k, rnd & 1);
#else
    if (jb < nplane) {
      static_for<JV_S - 1>([&](auto kc) {
        constexpr int K = decltype(kc)::value;
        if (jb + K < nplane) step(jb + K, K, rnd & 1);
      });
    }
#endif
    // release the stages this warp did not compute on: the last staged plane (read only as
    // a z + 1 neighbour) and the padding of the segment's last round
    const int npad = (nplane + 1 + JV_S - 1) / JV_S * JV_S;
    __syncwarp();
    if (threadIdx.x == 0)
      for (int j = nplane; j < npad; ++j) {
        // an empty stage is released only once the producer has opened it: a warp must not
        // arrive twice in one phase of an empty barrier (two short segments in a row)
        if (j > nplane) mbar_wait(full0 + 8 * (j % JV_S), (r0 + j / JV_S) & 1);
        mbar_arrive(empty0 + 8 * (j % JV_S));
      }
    rnd = r0 + npad / JV_S;
    u += zb - za;
  }
  if constexpr (DOT) {   // CTA partials of the fused dot products (fixed order; compute warps only)
    __shared__ double dsh[2][T_WARPS];
    for (int o = 16; o > 0; o >>= 1) {
      dacc1 += __shfl_down_sync(0xffffffffu, dacc1, o);
      dacc2 += __shfl_down_sync(0xffffffffu, dacc2, o);
    }
    if (threadIdx.x == 0) {
      dsh[0][threadIdx.y] = dacc1;
      dsh[1][threadIdx.y] = dacc2;
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(T_WARPS * VX) : "memory");   // the producer warp has left
    if (tid == 0) {
      double a1 = 0.0, a2 = 0.0;
      for (int k = 0; k < T_WARPS; ++k) {
        a1 += dsh[0][k];
        a2 += dsh[1][k];
      }
      F.dot_part[blockIdx.x] = a1;
      if (F.dot_two) F.dot_part[gridDim.x + blockIdx.x] = a2;
    }
  }
}

// CTAs of the persistent J v: one resident wave (the smallest occupancy of the four
// instantiations), at least min_planes_per_cta() units per CTA on small grids
template <bool OC, bool DOT>
inline int jv_per_sm() {
  static int per_sm = 0;
  if (!per_sm) {
    using L = JvLayout;
    const size_t smem = (size_t)JV_S * L::SLOT + 128 + 16 * JV_S;   // ring + alignment slack + mbarriers
    auto kern = k_jv_tma<OC, DOT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::THREADS, smem);
    if (per_sm < 1) per_sm = 1;
  }
  return per_sm;
}
inline int jv_grid_size(int n_sm, long long units) {
  const int per_sm = std::min(std::min(jv_per_sm<true, true>(), jv_per_sm<true, false>()),
                              std::min(jv_per_sm<false, true>(), jv_per_sm<false, false>()));
  const long long g = std::min<long long>((long long)per_sm * n_sm, units / min_planes_per_cta());
  return (int)std::max<long long>(g, 1);
}

// launches the persistent J v; false if the grid or the pointers do not allow tensor-map tiles
inline bool jv_launch_tma(TmaCache& cache, const DevParams& P, const FineArgs& F, const int32_t* labt,
                          const double2* V, double inv_dt, int flags, double2* out2, const int32_t* bounds,
                          int n_cta, cudaStream_t s) {
  using L = JvLayout;
  if (!tma_grid_ok(P) || !labt || !bounds || n_cta < 1) return false;
  TmaMaps M;
  std::memset(&M, 0, sizeof(M));
  const CUtensorMap* m = tma_map(cache, labt, 3, P.nx, P.ny, P.nz);
  if (!m) return false;
  M.lab = *m;
  if (!(m = tma_map(cache, V, 1, P.nx, P.ny, P.nz))) return false;
  M.val = *m;
  const bool oc = flags & 4;
  if (oc) {
    if (!(m = tma_map(cache, F.w, 2, P.nx, P.ny, P.nz))) return false;
    M.aux = *m;
  }
  const size_t smem = (size_t)JV_S * L::SLOT + 128 + 16 * JV_S;   // ring + alignment slack + mbarriers
  const int tbx = (P.nx + VX - 1) / VX, tby = (P.ny + VY - 1) / VY;
  if (F.dot_nblk) *F.dot_nblk = n_cta;
  auto go = [&](auto onec, auto dotc) {
    constexpr bool OC = decltype(onec)::value, DOT = decltype(dotc)::value;
    jv_per_sm<OC, DOT>();   // function attributes
    launch(k_jv_tma<OC, DOT>, dim3((unsigned)n_cta), dim3(VX, L::THREADS / VX, 1), smem, s, P, M, F, labt, V,
           inv_dt, flags, out2, tbx, tby, bounds);
  };
  if (oc) {
    if (F.dot_a) go(std::true_type{}, std::true_type{});
    else go(std::true_type{}, std::false_type{});
  } else {
    if (F.dot_a) go(std::false_type{}, std::true_type{});
    else go(std::false_type{}, std::false_type{});
  }
  return true;
}

}  // namespace hc
