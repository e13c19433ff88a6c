// TMA-fed 2.5-D stencil: the solver's matrix-free J v and fine-level multigrid
// sweeps on grids whose x pitch allows tensor-map tiles (nx % 4 == 0).
//
// A CTA owns a 32 x 8 column of the grid and marches zc planes.  Every plane's tile
// plus its one-voxel x/y halo is brought into a 4-deep shared-memory ring by ONE
// thread with cp.async.bulk.tensor (labels 40 x 10 int32, values 34 x 10 double2 or
// 36 x 10 double, gX/c 36 x 10 double), completion signalled on a per-slot mbarrier; the
// other 255 threads issue no load instructions for the stencil operands at all.
// Out-of-domain halo elements (x/y edges, plane -1 and plane nz) are zero-filled by
// the TMA unit: label 0 is the "void" phase whose face coefficients are zero, so
// missing neighbours contribute nothing — the reference's face enumeration
// (operator.py:121-242) without a single boundary branch.
//
// Face word (labt, below): phase, interface and same-phase conduction masks, and the
// tile-plane-local first face slot, 0 = outside; the slots hold row-oriented
// (alpha, beta, gamma) triples (cslot).  The contact-face table is indexed (a << 3) | b.
#pragma once

#include <cuda.h>

#include <cstring>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "hc_stencil.cuh"

namespace hc {

// phases in the TMA label encoding
enum : int { TV = 0, TEL = EL + 1, TGR = GR + 1, TCC = CC + 1, TCW = CW + 1 };
// face word (one int32 per voxel, built once per geometry):
//   (phase + 1) | interface mask << 3 | same-phase conduction mask << FW_SELF |
//   contact flag | grounded-row flag | tile-plane-local first face slot << FW_SLOT
// Direction bits: 0 x-1, 1 x+1, 2 y-1, 3 y+1, 4 z-1, 5 z+1.  The conduction mask holds the
// in-domain neighbours of the same phase (kind K_CONT): their faces use the row phase's own
// (P, C), so the stencil reads no neighbour label and no pair table.  A voxel with a
// contact face (two different conductor phases, harmonic-mean conductance) takes the
// table path on all its faces.
constexpr int FW_SELF = 9, FW_SLOT = 17;
constexpr int FW_CONTACT = 1 << 15, FW_GROUND = 1 << 16;
// operator value (residual) mode of the TMA stencil: parts in `flags`, mu in `omega`,
// c_prev in `r`, interface currents per face slot in F.islot
constexpr int SM_RES = 4;

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load3(unsigned dst, const CUtensorMap* map, int x, int y, int z,
                                          unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
               : "memory");
}

// tensor maps of one launch (passed by value; __grid_constant__ keeps them in param space)
struct TmaMaps {
  CUtensorMap lab;   // int32 [nz][ny][nx], box 40 x 10 x 1
  CUtensorMap val;   // values: double2 as float64 [nz][ny][2 nx] box 68 x 10, or double box 36 x 10
  CUtensorMap aux;   // gX/c (FULL) or r (SMOOTH0), double box 36 x 10
  CUtensorMap aux2;  // dinv (SMOOTH0)
};

#ifndef HC_TMA_STAGES
#define HC_TMA_STAGES 4
#endif
constexpr int T_S = HC_TMA_STAGES;   // ring depth
#ifndef HC_TMA_MINB
#define HC_TMA_MINB 3
#endif
#ifndef HC_TMA_DOTPF
#define HC_TMA_DOTPF 0   // planes of L2 prefetch distance for the fused dot operand (0: off; measured +1 % step rate, -1 % standalone J v)
#endif

template <typename Fn, int... I>
__device__ __forceinline__ void static_for_impl(Fn&& fn, std::integer_sequence<int, I...>) {
  (fn(std::integral_constant<int, I>{}), ...);
}
template <int N, typename Fn>
__device__ __forceinline__ void static_for(Fn&& fn) {
  static_for_impl(fn, std::make_integer_sequence<int, N>{});
}
constexpr int T_TH = VY + 2;
// TMA box starts must be 16-byte aligned in x, so each tile starts at the aligned
// column at or below x0 - 1:  int32 labels at x0 - 4 (40 wide), double tiles at
// x0 - 2 (36 wide), double2 tiles at x0 - 1 (34 wide).
constexpr int T_LW = VX + 8, T_LOFF = 4;    // labels
constexpr int T_DW = VX + 4, T_DOFF = 2;    // double (scalar values, gX/c, r, dinv)
constexpr int T_QW = VX + 2, T_QOFF = 1;    // double2 values
constexpr int T_LN = T_LW * T_TH, T_DN = T_DW * T_TH, T_QN = T_QW * T_TH;
// interface face slots staged per (tile, plane): up to T_SLOTCAP 32-byte slots (the rest,
// on very interface-dense tile-planes, is read from global memory)
#ifndef HC_TMA_SLOTCAP
#define HC_TMA_SLOTCAP 256
#endif
constexpr int T_SLOTCAP = HC_TMA_SLOTCAP;

template <int MODE, int EPI>
struct TmaLayout {
  static constexpr bool FULLM = MODE == SM_FULL || MODE == 4;   // double2 (c, phi) tiles
  static constexpr bool X0 = EPI == EP_SMOOTH0 || EPI == EP_RESID0;
  static constexpr int VW = FULLM ? T_QW : T_DW, VOFF = FULLM ? T_QOFF : T_DOFF;
  static constexpr int VBYTES = FULLM ? T_QN * 16 : T_DN * 8;
  static constexpr int LAB = 0;                                         // int32 [T_LN]
  static constexpr int VAL = ((T_LN * 4 + 127) / 128) * 128;            // value tile
  static constexpr int AUX = VAL + (X0 ? 0 : ((VBYTES + 127) / 128) * 128);   // gX/c or r
  static constexpr bool HAS_AUX = FULLM || X0;
  static constexpr int AUX2 = AUX + (HAS_AUX ? ((T_DN * 8 + 127) / 128) * 128 : 0);
  static constexpr int LOG = AUX2 + (X0 ? ((T_DN * 8 + 127) / 128) * 128 : 0);   // log c (residual)
  static constexpr int SLT = LOG + (MODE == 4 ? ((T_QN * 8 + 127) / 128) * 128 : 0);  // face slots
  static constexpr bool HAS_SLT = true;
  static constexpr int SB = MODE == 4 ? 8 : 32;   // bytes per staged slot: current | (alpha, beta, gamma, pad)
  static constexpr int SLOT = SLT + ((T_SLOTCAP + 2) * SB + 127) / 128 * 128;
  static constexpr int THREADS = VX * (VY + 1);   // + producer warp
};

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// Warp-specialised: warps 0..7 compute (one voxel per thread and plane), warp 8 is
// the producer.  full[s] completes when plane s's tiles have landed (TMA transaction
// bytes), empty[s] when all eight compute warps are done with it, so compute warps
// drift freely within the ring instead of meeting at a CTA barrier every plane.
constexpr int T_WARPS = VY;                 // compute warps
constexpr int T_THREADS = VX * (VY + 1);    // + producer warp

template <int MODE, int EPI, bool ONEC>
__global__ void __launch_bounds__(TmaLayout<MODE, EPI>::THREADS, HC_TMA_MINB)
k_fine_tma(DevParams P, const __grid_constant__ TmaMaps M, FineArgs F, const int32_t* __restrict__ labt,
           const double2* __restrict__ V, const double* __restrict__ e, const double* __restrict__ r,
           const double* __restrict__ dinv, double omega, double inv_dt, int flags,
           double2* __restrict__ out2, double* __restrict__ out, int zc, int zb, int ze) {
  using L = TmaLayout<MODE, EPI>;
  constexpr bool FULLM = L::FULLM, X0 = L::X0;
  constexpr bool RES = MODE == SM_RES;
  constexpr bool OC = MODE == SM_FULL && ONEC;
  using VT = typename std::conditional<FULLM, double2, double>::type;
  extern __shared__ __align__(16) unsigned char smem_dyn[];
  // 128-byte aligned ring (the launch adds 128 bytes of slack)
  unsigned char* ring = smem_dyn + ((128 - ((unsigned)__cvta_generic_to_shared(smem_dyn) & 127)) & 127);
  __shared__ __align__(16) double2 sPC[64];   // (P, C) per (a << 3 | b): contact voxels
  __shared__ __align__(16) double2 sSelf[8];  // (P, C) of a phase's same-phase faces, per a
  __shared__ __align__(8) unsigned long long full[T_S], empty[T_S], ready[T_S];
  __shared__ int tp_start[T_S];   // first global face slot of the tile-plane staged in each ring slot
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  const int x0 = blockIdx.x * VX, y0 = blockIdx.y * VY;
  // planes zb .. ze - 1 are computed (the whole grid, or the z range holding the field's rows)
  const int z0 = zb + blockIdx.z * zc, z1 = min(z0 + zc, ze);   // planes z0 .. z1 are staged
  const int nplane = z1 - z0;                                // computed planes
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(full);
  const unsigned empty0 = (unsigned)__cvta_generic_to_shared(empty);
  const unsigned ready0 = (unsigned)__cvta_generic_to_shared(ready);
  const int tid = threadIdx.y * VX + threadIdx.x;
  if (tid == T_WARPS * VX) {
#pragma unroll
    for (int k = 0; k < T_S; ++k) {
      mbar_init(full0 + 8 * k, 1);
      mbar_init(empty0 + 8 * k, T_WARPS);
      if constexpr (RES) mbar_init(ready0 + 8 * k, T_WARPS);
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
  // producer warp: face-slot block of plane j = lane + 32 r of this tile column (loaded
  // lane-parallel; the first batch before the barrier so its latency overlaps the setup)
  int st_l = 0, cnt_l = 0;
  auto load_tp = [&](int jb) {
    st_l = cnt_l = 0;
    const int zz = z0 + jb + (int)threadIdx.x;
    if (L::HAS_SLT && jb + (int)threadIdx.x <= nplane && zz < nz) {
      const long long tpi = ((long long)zz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      st_l = F.tp_off[tpi];
      cnt_l = min(F.tp_off[tpi + 1] - st_l, T_SLOTCAP);
    }
  };
  if (threadIdx.y == T_WARPS) load_tp(0);
  __syncthreads();   // barriers initialised, tables built (the only CTA-wide barrier)
  // programmatic dependent launch: everything above reads only static data (parameters,
  // slot offsets), so it overlaps the predecessor kernel's tail; operands come after this
  pdl_wait();

  if (threadIdx.y == T_WARPS) {   // ---------------- producer warp
    const int lane = threadIdx.x;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(ring);
    constexpr unsigned tx = T_LN * 4 + (X0 ? 2 * T_DN * 8 : L::VBYTES);
    // gX/c tiles only on planes next to electrolyte in this tile column (it is zero
    // elsewhere and only electrolyte rows read it)
    int2 elz = make_int2(0, -1);
    if constexpr (OC) elz = F.elz[blockIdx.y * gridDim.x + blockIdx.x];
    for (int j = 0; j <= nplane; ++j) {
      if (j && (j & 31) == 0) load_tp(j);
      const int st = __shfl_sync(0xffffffffu, st_l, j & 31), cnt = __shfl_sync(0xffffffffu, cnt_l, j & 31);
      if (lane == 0) {
        const int slot = j % T_S;
        if (j >= T_S) mbar_wait(empty0 + 8 * slot, ((j / T_S) - 1) & 1);
        const unsigned b = full0 + 8 * slot, s = sbase + slot * L::SLOT;
        const int zz = z0 + j;
        const bool wtile = OC && zz >= elz.x - 1 && zz <= elz.y + 1;
        // residual slots are 8 B: start the bulk copy at the 16-byte aligned slot below
        const int sta = RES ? (st & ~1) : st;
        const unsigned sbytes = RES ? (unsigned)(((cnt + (st - sta)) * 8 + 15) & ~15) : 32u * cnt;
        tp_start[slot] = st;   // true first slot (the residual copy starts at the 16-byte aligned sta)
        mbar_expect_tx(b, tx + (wtile ? T_DN * 8 : 0) + (cnt ? sbytes : 0u));
        tma_load3(s + L::LAB, &M.lab, x0 - T_LOFF, y0 - 1, zz, b);
        if constexpr (X0) {
          tma_load3(s + L::AUX, &M.aux, x0 - T_DOFF, y0 - 1, zz, b);
          tma_load3(s + L::AUX2, &M.aux2, x0 - T_DOFF, y0 - 1, zz, b);
        } else if constexpr (FULLM) {
          tma_load3(s + L::VAL, &M.val, 2 * (x0 - T_QOFF), y0 - 1, zz, b);
          if (wtile) tma_load3(s + L::AUX, &M.aux, x0 - T_DOFF, y0 - 1, zz, b);
        } else {
          tma_load3(s + L::VAL, &M.val, x0 - T_DOFF, y0 - 1, zz, b);
        }
        if (cnt) {
          if constexpr (RES) bulk_load(s + L::SLT, F.islot + sta, sbytes, b);
          else bulk_load(s + L::SLT, F.cslot + 4LL * st, sbytes, b);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------- compute warps
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  const bool active = x < nx && y < ny;
  const int col = active ? y * nx + x : 0;
  VT vm{};            // own column z - 1 (registers)
  double wm = 0.0;   // gX/c (J v) or log c (residual) of the own column at z - 1
  int lm = 0;
  if (active && z0 > 0) {
    const long long idx = (long long)(z0 - 1) * nxy + col;
    lm = labt[idx] & 7;
    if constexpr (FULLM) {
      vm = V[idx];
      if constexpr (OC) wm = F.w[idx];
      if constexpr (RES) wm = (lm == TEL) ? log(vm.x) : 0.0;
    } else if constexpr (X0) {
      vm = omega * dinv[idx] * r[idx];
    } else {
      vm = e[idx];
    }
  }
  const double tp = P.t_plus;
  constexpr int VW = X0 ? T_DW : L::VW;
  // byte offsets of the own voxel inside a slot
  const int lofs = L::LAB + 4 * ((threadIdx.y + 1) * T_LW + threadIdx.x + T_LOFF);
  const int aofs = 8 * ((threadIdx.y + 1) * T_DW + threadIdx.x + T_DOFF);
  const int vofs = X0 ? aofs : L::VAL + (int)sizeof(VT) * ((threadIdx.y + 1) * L::VW + threadIdx.x + L::VOFF);
  const unsigned char* base = ring;
  const int vidx_t = (threadIdx.y + 1) * T_QW + threadIdx.x + T_QOFF;   // own element of a double2-shaped tile

  // residual: log c of the staged electrolyte elements of plane p, computed cooperatively
  // by the eight compute warps two planes ahead (each tile element once instead of once
  // per electrolyte face); ready[s] completes when all warps have written their share
  auto logs_for = [&](int p) {
    if (p > nplane) return;
    const int slot = p % T_S;
    mbar_wait(full0 + 8 * slot, (p / T_S) & 1);
    unsigned char* S = ring + slot * L::SLOT;
    for (int i = threadIdx.y * VX + threadIdx.x; i < T_QN; i += T_WARPS * VX) {
      const int row = i / T_QW, c = i - row * T_QW;
      const int lab = reinterpret_cast<const int*>(S + L::LAB)[row * T_LW + c + (T_LOFF - T_QOFF)];
      if ((lab & 7) == TEL)
        reinterpret_cast<double*>(S + L::LOG)[i] = log(reinterpret_cast<const double2*>(S + L::VAL)[i].x);
    }
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(ready0 + 8 * slot);
  };
  if constexpr (RES) {
    logs_for(0);
    logs_for(1);
  }
  auto lab_at = [&](const unsigned char* Sx, int o) -> int {
    return *reinterpret_cast<const int*>(Sx + lofs + 4 * o);
  };
  auto val_at = [&](const unsigned char* Sx, int o) -> VT {
    if constexpr (X0)
      return omega * *reinterpret_cast<const double*>(Sx + L::AUX2 + aofs + 8 * o) *
             *reinterpret_cast<const double*>(Sx + L::AUX + aofs + 8 * o);
    else
      return *reinterpret_cast<const VT*>(Sx + vofs + (int)sizeof(VT) * o);
  };
  auto w_at = [&](const unsigned char* Sx, int o) -> double {
    return *reinterpret_cast<const double*>(Sx + L::AUX + aofs + 8 * o);
  };
  auto lg = [&](const unsigned char* Sx, int o) -> double {
    return reinterpret_cast<const double*>(Sx + L::LOG)[vidx_t + o];
  };
  // the own voxel of plane z0; afterwards it is carried from the previous plane's z + 1 read
  int aw = 0;
  VT va{};
  double wa = 0.0;
  mbar_wait((RES ? ready0 : full0), 0);
  aw = lab_at(base, 0);
  va = val_at(base, 0);
  if constexpr (OC) wa = w_at(base, 0);
  if constexpr (RES) wa = lg(base, 0);

  double dacc1 = 0.0, dacc2 = 0.0;   // fused dot products (J v with F.dot_a)
  auto step = [&](int j, auto slotc, unsigned ph1) {
    constexpr int K = decltype(slotc)::value, K1 = (K + 1) % T_S;
    const unsigned char* S0 = base + K * L::SLOT;
    const unsigned char* S1 = base + K1 * L::SLOT;
    const int z = z0 + j;
    const int v = z * nxy + col;
    double rv = 0.0, dv_ = 0.0;
    if constexpr (!FULLM) {
      if (active) {
        if (EPI != EP_STORE) rv = r[v];
        if (EPI == EP_SMOOTH || EPI == EP_SMOOTH0) dv_ = dinv[v];
      }
    } else if constexpr (RES) {
      if (active && (flags & PART_TIME)) rv = r[v];   // c_prev
    }
    if constexpr (RES) logs_for(j + 2);
    if constexpr (MODE == SM_FULL) {
      // the fused dot products' second operand is the one per-thread global load of the plane
      // step (ncu: 37 % of the in-solver stall samples sat on its first use); ask L2 for the
      // line HC_TMA_DOTPF planes ahead
#if HC_TMA_DOTPF > 0
      if (F.dot_a && active && z + HC_TMA_DOTPF < nz)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(F.dot_a + v + (long long)HC_TMA_DOTPF * nxy));
#endif
    }
    // plane j was waited for as the previous step's z + 1
    mbar_wait((RES ? ready0 : full0) + 8 * K1, ph1);
    // own column at z + 1: the z + 1 neighbour now, the own voxel of the next plane
    const int aw1 = lab_at(S1, 0);
    const VT v1 = val_at(S1, 0);
    double w1 = 0.0;
    if constexpr (OC) w1 = w_at(S1, 0);
    if constexpr (RES) w1 = lg(S1, 0);
    // neighbour d: 0 x-1, 1 x+1, 2 y-1, 3 y+1, 4 z-1 (registers), 5 z+1 (registers)
    auto nb_lab = [&](int d) -> int {
      if (d == 4) return lm;
      if (d == 5) return aw1 & 7;
      return lab_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_LW : T_LW))) & 7;
    };
    auto nb_val = [&](int d) -> VT {
      if (d == 4) return vm;
      if (d == 5) return v1;
      return val_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -VW : VW)));
    };
    auto nb_w = [&](int d) -> double {
      if (d == 4) return wm;
      if (d == 5) return w1;
      return w_at(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_DW : T_DW)));
    };
    auto nb_lg = [&](int d) -> double {
      if (d == 4) return wm;
      if (d == 5) return w1;
      return lg(S0, d == 0 ? -1 : (d == 1 ? 1 : (d == 2 ? -T_QW : T_QW)));
    };
    const int a = aw & 7;
    if (active) {
      const bool in_row = (MODE == SM_CONC || MODE == SM_CP) ? (a == TGR || a == TEL) : !(aw & FW_GROUND);
      if (!in_row) {
        if constexpr (FULLM) out2[v] = make_double2(0.0, 0.0);
        else out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = 0.0;
      } else {
        const bool elrow = a == TEL;
        const unsigned sm = ((unsigned)aw >> FW_SELF) & 63u;   // same-phase conduction faces
        double rc = 0.0, rp = 0.0;
        if (aw & FW_CONTACT) {
          // rare (solid conductors touching another conductor phase): the (P, C) table of
          // the face's phase pair on every face.  Never an electrolyte row.
          const int a8 = a << 3;
          const bool lin = !RES || (flags & PART_LIN);
#pragma unroll
          for (int d = 0; d < 6; ++d) {
            const double2 pc = sPC[a8 | nb_lab(d)];
            const VT vbd = nb_val(d);
            if constexpr (FULLM) {
              if (lin) {
                rp = fma(pc.x, va.y - vbd.y, rp);
                rc = fma(pc.y, va.x - vbd.x, rc);
              }
            } else if (MODE == SM_PHI || MODE == SM_CONC) {
              rp = fma(MODE == SM_PHI ? pc.x : pc.y, va - vbd, rp);
            }
          }
        } else {
          // same-phase faces share the row phase's coefficients: sum the differences
          // over the conduction mask, scale once.  Electrolyte rows also carry migration
          // and chemical-potential couplings, which equal t+ times their phi-row terms
          // (operator.py:216-227), so only P and C are needed.
          const double2 ps = sSelf[a];
          if constexpr (RES) {
            // linear two-point fluxes and the chemical-potential faces gX (log c_a - log c_b)
            // between electrolyte voxels (operator.py:322-327)
            double dp = 0.0, dc = 0.0, q = 0.0;
#pragma unroll
            for (int d = 0; d < 6; ++d)
              if (sm & (1u << d)) {
                const double2 vbd = nb_val(d);
                dp += va.y - vbd.y;
                dc += va.x - vbd.x;
                q += wa - nb_lg(d);
              }
            if (flags & PART_LIN) {
              rp = ps.x * dp;
              rc = ps.y * dc;
            }
            if ((flags & PART_1C) && elrow) rp = fma(P.gX, q, rp);
          } else if constexpr (FULLM) {
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
          } else if (MODE == SM_PHI || MODE == SM_CONC) {
            double dq = 0.0;
#pragma unroll
            for (int d = 0; d < 6; ++d)
              if (sm & (1u << d)) dq += va - nb_val(d);
            rp = (MODE == SM_PHI ? ps.x : ps.y) * dq;
          }
        }
        // interface kinetics: the voxel's face slots, consecutive in direction order from the
        // tile-plane-local index in its word (staged with the plane; global past capacity)
        double si = 0.0;
        const unsigned mask = ((unsigned)aw >> 3) & 63u;
        if (mask) {
          const int loc = (int)((unsigned)aw >> FW_SLOT), n = __popc(mask);
          if constexpr (RES) {
            // interface currents, one per face slot, oriented from this row (k_residual_islot)
            if (flags & PART_BV) {
              if (loc + n <= T_SLOTCAP) {
                const double* c = reinterpret_cast<const double*>(S0 + L::SLT) + loc + (tp_start[K] & 1);
                for (int k = 0; k < n; ++k) si += c[k];
              } else {
                const double* c = F.islot + tp_start[K] + loc;
                for (int k = 0; k < n; ++k) si += c[k];
              }
            }
          } else {
            // face d adds alpha c_a + beta c_b + gamma (phi_a - phi_b) to the phi row
            auto faces = [&](const double* c) {
#pragma unroll
              for (int d = 0; d < 6; ++d) {
                if (mask & (1u << d)) {
                  const double2 ab = *reinterpret_cast<const double2*>(c);
                  const double g = c[2];
                  const VT vbd = nb_val(d);
                  if constexpr (FULLM) si += ab.x * va.x + ab.y * vbd.x + g * (va.y - vbd.y);
                  else if (MODE == SM_CONC) si += ab.x * va + ab.y * vbd;
                  else si += g * (va - vbd);
                  c += 4;
                }
              }
            };
            if (loc + n <= T_SLOTCAP) faces(reinterpret_cast<const double*>(S0 + L::SLT) + 4 * loc);
            else faces(F.cslot + 4LL * (tp_start[K] + loc));
          }
        }
        if constexpr (RES) {
          const bool crow = a == TGR || elrow;
          if (elrow) rc = fma(tp, rp, rc);   // migration + chemical potential: t+ x phi-row terms
          if (crow) rc += si;
          rp += si;
          if ((flags & PART_BND) && a == TCW && z == 0) rp = fma(omega, P.drive, rp);
          if ((flags & PART_TIME) && crow) rc += (va.x - rv) * inv_dt;
          out2[v] = make_double2(rc, rp);
        } else if constexpr (FULLM) {
          const bool crow = a == TGR || elrow;
          if (elrow) rc = (flags & 2) ? fma(1.0 - tp, si, rc) : fma(tp, rp, rc) + si;  // T: c -= t+ phi
          else if (crow) rc += si;
          rp += si;
          if ((flags & 1) && crow) rc = fma(va.x, inv_dt, rc);
          if (flags & 8) rc = 0.0;
          out2[v] = make_double2(rc, rp);
          if (MODE == SM_FULL && F.dot_a) {
            const double2 da = F.dot_a[v];
            dacc1 += rc * da.x + rp * da.y;
            dacc2 += rc * rc + rp * rp;
          }
        } else {
          if (MODE == SM_PHI) rp += si;
          else rp = fma(elrow ? 1.0 - tp : 1.0, si, rp);   // (T J) on electrolyte c rows
          if (MODE == SM_CONC) rp = fma(inv_dt, va, rp);
          if (EPI == EP_STORE) out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = rp;
          else if (EPI == EP_RESID || EPI == EP_RESID0) out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = rv - rp;
          else out[(size_t)v * ((flags & FL_OSTRIDE2) ? 2 : 1)] = va + omega * dv_ * (rv - rp);
        }
      }
      if constexpr (EPI == EP_RESID0) reinterpret_cast<double*>(out2)[v] = va;
    }
    lm = a;
    vm = va;
    if constexpr (OC || RES) wm = wa;
    aw = aw1;
    va = v1;
    wa = w1;
    __syncwarp();
    if (threadIdx.x == 0) mbar_arrive(empty0 + 8 * K);   // this warp is done with plane j
  };
  for (int jb = 0; jb < nplane; jb += T_S) {   // unrolled by the ring depth: slots are compile-time
    const unsigned ph = (jb / T_S) & 1;
    static_for<T_S>([&](auto kc) {
      constexpr int K = decltype(kc)::value;
      if (jb + K < nplane) step(jb + K, kc, K + 1 == T_S ? ph ^ 1 : ph);
    });
  }
  if constexpr (MODE == SM_FULL) {
    if (F.dot_a) {   // CTA partials of the fused dot products (fixed order; compute warps only)
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
        const int nb = gridDim.x * gridDim.y * gridDim.z;
        const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        F.dot_part[b] = a1;
        if (F.dot_two) F.dot_part[nb + b] = a2;
      }
    }
  }
}

// ---- host side: tensor-map encoding (driver entry point, no -lcuda) and a cache
// keyed by (pointer, element kind) so graph captures and repeated launches reuse maps.
struct TmaCache {
  std::mutex mu;
  std::unordered_map<unsigned long long, CUtensorMap> maps;
};

bool tma_encode(CUtensorMap* m, const void* ptr, int kind, int nx, int ny, int nz);
// kind: 0 int32 labels (box 40), 1 double2 values (box 68 f64), 2 double (box 36)
inline const CUtensorMap* tma_map(TmaCache& c, const void* ptr, int kind, int nx, int ny, int nz) {
  const unsigned long long key = reinterpret_cast<unsigned long long>(ptr) ^ ((unsigned long long)kind << 60);
  std::lock_guard<std::mutex> g(c.mu);
  auto it = c.maps.find(key);
  if (it != c.maps.end()) return &it->second;
  // transient buffers (e.g. per-call tensors of the Python API) would grow the cache
  // without bound; maps are cheap to re-encode, so start over past a few thousand
  if (c.maps.size() >= 4096) c.maps.clear();
  CUtensorMap m;
  if (!tma_encode(&m, ptr, kind, nx, ny, nz)) return nullptr;
  return &c.maps.emplace(key, m).first->second;
}

inline bool tma_grid_ok(const DevParams& P) { return P.nx % 4 == 0 && P.nx >= 4; }

template <int MODE, int EPI>
inline bool fine_launch_tma(TmaCache& cache, const DevParams& P, const FineArgs& F, const int32_t* labt,
                            const double2* V, const double* e, const double* r, const double* dinv,
                            double omega, double inv_dt, int flags, double2* out2, double* out,
                            int n_sm, cudaStream_t s) {
  using L = TmaLayout<MODE, EPI>;
  if (!tma_grid_ok(P) || !labt) return false;
  TmaMaps M;
  std::memset(&M, 0, sizeof(M));
  const CUtensorMap* m = tma_map(cache, labt, 0, P.nx, P.ny, P.nz);
  if (!m) return false;
  M.lab = *m;
  if constexpr (L::X0) {
    if (!(m = tma_map(cache, r, 2, P.nx, P.ny, P.nz))) return false;
    M.aux = *m;
    if (!(m = tma_map(cache, dinv, 2, P.nx, P.ny, P.nz))) return false;
    M.aux2 = *m;
  } else if constexpr (L::FULLM) {
    if (!(m = tma_map(cache, V, 1, P.nx, P.ny, P.nz))) return false;
    M.val = *m;
    if (MODE == SM_FULL && (flags & 4)) {
      if (!(m = tma_map(cache, F.w, 2, P.nx, P.ny, P.nz))) return false;
      M.aux = *m;
    }
  } else {
    if (!(m = tma_map(cache, e, 2, P.nx, P.ny, P.nz))) return false;
    M.val = *m;
  }
  const size_t smem = (size_t)T_S * L::SLOT + 128;
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  auto go = [&](auto onec) {
    constexpr bool OC = decltype(onec)::value;
    auto kern = k_fine_tma<MODE, EPI, OC>;
    static int per_sm = 0;   // one per (MODE, EPI, OC) instantiation
    if (!per_sm) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::THREADS, smem);
      if (per_sm < 1) per_sm = 1;
    }
    // the c-block modes sweep only the planes that hold c rows (F.cz; the buffers they write
    // are zero outside and stay so: nothing else ever writes those entries)
    const bool crange = (MODE == SM_CONC || MODE == SM_CP) && F.cz.y > F.cz.x;
    const int zb = crange ? F.cz.x : 0, ze = crange ? F.cz.y : P.nz, nzr = ze - zb;
    const int bz = pick_bz(bx, by, nzr, per_sm, n_sm);
    const int zc = (nzr + bz - 1) / bz;
    const dim3 grid(bx, by, (nzr + zc - 1) / zc);
    if (F.dot_nblk) *F.dot_nblk = (int)(grid.x * grid.y * grid.z);
    launch(kern, grid, dim3(VX, L::THREADS / VX, 1), smem, s, P, M, F, labt,
           V, e, r, dinv, omega, inv_dt, flags, out2, out, zc, zb, ze);
  };
  if (MODE == SM_FULL && (flags & 4)) go(std::true_type{});
  else go(std::false_type{});
  return true;
}

// residual through the TMA stencil (parts bitmask PART_*); false if the grid or the
// pointers do not allow tensor-map tiles
inline bool res_launch_tma(Operator& op, const double2* X, double mu, int parts, const double* cprev,
                           double inv_dt, double2* out, cudaStream_t s) {
  if (op.stencil_kind != 3 || !op.tma) return false;
  FineArgs F{op.labels.p, op.if_rank.p, op.if_vcoef.p, (long long)op.if_dir.n, op.inv_c.p,
             op.if_cslot.p, op.elz.p, op.if_islot.p, op.tp_off.p};
  return fine_launch_tma<SM_RES, EP_STORE>(*op.tma, op.P, F, op.labt.p, X, nullptr, cprev, nullptr, mu,
                                           inv_dt, parts, out, nullptr, op.n_sm, s);
}

// the solver's dispatcher: TMA ring where the grid allows it, else the cp.async ring
template <int MODE, int EPI>
inline void fine_launch_op(Operator& op, const FineArgs& F, const double2* V, const double* e,
                           const double* r, const double* dinv, double omega, double inv_dt, int flags,
                           double2* out2, double* out, cudaStream_t s) {
  if (op.stencil_kind == 3 && op.tma &&
      fine_launch_tma<MODE, EPI>(*op.tma, op.P, F, op.labt.p, V, e, r, dinv, omega, inv_dt, flags, out2,
                                 out, op.n_sm, s))
    return;
  fine_launch_p<MODE, EPI>(op.P, F, op.lab4.p, V, e, r, dinv, omega, inv_dt, flags, out2, out, op.n_sm, s);
}

}  // namespace hc
