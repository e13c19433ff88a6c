// Register-blocked TMA stencil for the matrix-free J v (the Krylov operator).
//
// Same TMA ring and 32 x 8 tiles as k_fine_tma (hc_tma.cuh): one producer warp stages
// every plane's labels, (c, phi) values, gX/c and interface face slots with
// cp.async.bulk(.tensor) into a 4-deep shared-memory ring.  The compute side differs:
// each compute thread owns YB consecutive y rows of one x column and marches z, and
// every face is evaluated ONCE and applied to both of its voxels:
//   * y faces between a thread's own rows: registers only;
//   * z faces: the face (z, z+1) is computed at plane z from the own rows of plane z+1,
//     its negative is carried in registers into plane z+1's accumulators, and plane z+1's
//     values become the next step's own values (each plane's own rows are read from
//     shared memory once, instead of once as "z+1" and again as "own");
//   * x faces: lane x computes (x, x+1) from lane x+1's values (warp shuffles) and hands
//     the negated flux back to lane x+1 (lane 31 / lane 0 use the tile's x halo);
//   * y faces to the rows of the neighbouring warp / tile: from the staged tile (halo).
// Compared with one voxel per thread re-reading its six neighbours from shared memory,
// this cuts the shared-memory wavefronts per voxel about in half and the face-table
// lookups from six to three, which is what bounded k_fine_tma<SM_FULL> (L1/TEX 74 % busy).
//
// Row semantics are those of k_fine_tma<SM_FULL> (operator.py:121-242 linear faces,
// 322-327 chemical-potential faces, 402-471 interface linearization): phi rows sum
// P(a,b)(phi_a - phi_b) plus, between electrolyte voxels, gX/c_a c_a - gX/c_b c_b; c rows
// sum C(a,b)(c_a - c_b), electrolyte c rows add t+ x their phi-row terms (or, under the
// row transform T, (1 - t+) x the interface terms); interface faces add the row-oriented
// alpha c_a + beta c_b + gamma (phi_a - phi_b); mass inv_dt on c rows.
#pragma once

#include "hc_tma.cuh"

namespace hc {

template <int YB>
struct YLayout {
  static constexpr int NW = VY / YB;          // compute warps
  static constexpr int THREADS = VX * (NW + 1);
  static constexpr int MINB = YB == 1 ? HC_TMA_MINB : 1;   // 3 CTAs per SM (the ring's shared memory allows 3)
};

template <int YB, bool OC>
__global__ void __launch_bounds__(YLayout<YB>::THREADS, YLayout<YB>::MINB)
k_jv_y(DevParams P, const __grid_constant__ TmaMaps M, FineArgs F, const int32_t* __restrict__ labt,
       const double2* __restrict__ V, double inv_dt, int flags, double2* __restrict__ out2, int zc) {
  using L = TmaLayout<SM_FULL, EP_STORE>;
  constexpr int NW = YLayout<YB>::NW;
  extern __shared__ __align__(16) unsigned char smem_dyn[];
  unsigned char* ring = smem_dyn + ((128 - ((unsigned)__cvta_generic_to_shared(smem_dyn) & 127)) & 127);
  __shared__ __align__(16) double2 sPC[64];
  __shared__ __align__(8) unsigned long long full[T_S], empty[T_S];
  __shared__ int tp_start[T_S];
  const int nx = P.nx, ny = P.ny, nz = P.nz, nxy = (int)P.nxy;
  const int x0 = blockIdx.x * VX, y0 = blockIdx.y * VY;
  const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
  const int nplane = z1 - z0;
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(full);
  const unsigned empty0 = (unsigned)__cvta_generic_to_shared(empty);
  const int warp = threadIdx.y, lane = threadIdx.x;
  const int tid = warp * VX + lane;
  if (tid == NW * VX) {
#pragma unroll
    for (int k = 0; k < T_S; ++k) {
      mbar_init(full0 + 8 * k, 1);
      mbar_init(empty0 + 8 * k, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 64) {
    const int a = tid >> 3, b = tid & 7;
    const bool ok = a >= 1 && a <= N_PHASES && b >= 1 && b <= N_PHASES;
    const int i = (a - 1) * 6 + (b - 1);
    sPC[tid] = ok ? make_double2(P.gP[i], P.gC[i]) : make_double2(0.0, 0.0);
  }
  int st_l = 0, cnt_l = 0;
  auto load_tp = [&](int jb) {
    st_l = cnt_l = 0;
    const int zz = z0 + jb + lane;
    if (jb + lane <= nplane && zz < nz) {
      const long long tpi = ((long long)zz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      st_l = F.tp_off[tpi];
      cnt_l = min(F.tp_off[tpi + 1] - st_l, T_SLOTCAP);
    }
  };
  if (warp == NW) load_tp(0);
  __syncthreads();
  pdl_wait();

  if (warp == NW) {   // ---------------- producer warp (as k_fine_tma<SM_FULL>)
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(ring);
    constexpr unsigned tx = T_LN * 4 + L::VBYTES;
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
        tp_start[slot] = st;
        mbar_expect_tx(b, tx + (wtile ? T_DN * 8 : 0) + 32u * cnt);
        tma_load3(s + L::LAB, &M.lab, x0 - T_LOFF, y0 - 1, zz, b);
        tma_load3(s + L::VAL, &M.val, 2 * (x0 - T_QOFF), y0 - 1, zz, b);
        if (wtile) tma_load3(s + L::AUX, &M.aux, x0 - T_DOFF, y0 - 1, zz, b);
        if (cnt) bulk_load(s + L::SLT, F.cslot + 4LL * st, 32u * cnt, b);
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------- compute warps
  const int x = x0 + lane;
  const int ty0 = warp * YB;                 // first own tile row
  const double tp = P.t_plus;
  // shared-memory element indices of the own rows (tile row ty0 + i sits at smem row ty0 + i + 1)
  auto li = [&](int r) { return r * T_LW + lane + T_LOFF; };   // labels
  auto qi = [&](int r) { return r * T_QW + lane + T_QOFF; };   // double2 values
  auto di = [&](int r) { return r * T_DW + lane + T_DOFF; };   // gX/c
  auto LAB = [&](int slot) { return reinterpret_cast<const int*>(ring + slot * L::SLOT + L::LAB); };
  auto VAL = [&](int slot) { return reinterpret_cast<const double2*>(ring + slot * L::SLOT + L::VAL); };
  auto WV = [&](int slot) { return reinterpret_cast<const double*>(ring + slot * L::SLOT + L::AUX); };

  // face between row phase a (value va, gX/c wa) and neighbour b: (c flux, phi flux) added
  // to a's rows and subtracted from b's
  auto face = [&](int la, double2 va, double wa, int lb, double2 vb, double wb, double& fc, double& fp) {
    const double2 pc = sPC[((la & 7) << 3) | (lb & 7)];
    fp = pc.x * (va.y - vb.y);
    fc = pc.y * (va.x - vb.x);
    if (OC && (la & 7) == TEL && (lb & 7) == TEL) fp += fma(wa, va.x, -wb * vb.x);
  };

  double2 cur[YB], prv[YB];
  double wcur[YB];
  int lcur[YB];
  double rc[YB], rp[YB];   // accumulators of the current plane (carry of the z face included)
  // plane z0 - 1 (own rows, global) and plane z0 (own rows, ring slot 0)
  mbar_wait(full0, 0);
#pragma unroll
  for (int i = 0; i < YB; ++i) {
    const int r = ty0 + i + 1;
    cur[i] = VAL(0)[qi(r)];
    lcur[i] = LAB(0)[li(r)];
    wcur[i] = OC ? WV(0)[di(r)] : 0.0;
    rc[i] = rp[i] = 0.0;
    prv[i] = make_double2(0.0, 0.0);
    const int y = y0 + ty0 + i;
    if (z0 > 0 && x < nx && y < ny) {
      const long long idx = (long long)(z0 - 1) * nxy + (long long)y * nx + x;
      const int lp = labt[idx];
      prv[i] = V[idx];
      const double wp = (OC && (lp & 7) == TEL) ? F.w[idx] : 0.0;
      double fc, fp;
      face(lcur[i], cur[i], wcur[i], lp, prv[i], wp, fc, fp);
      rc[i] = fc;
      rp[i] = fp;
    }
  }
  double dacc1 = 0.0, dacc2 = 0.0;

  auto step = [&](int j, auto slotc, unsigned ph1) {
    constexpr int K = decltype(slotc)::value, K1 = (K + 1) % T_S;
    const int z = z0 + j;
    mbar_wait(full0 + 8 * K1, ph1);   // plane z + 1 (slot K was waited for as K1 one step ago)
    const int* L0 = LAB(K);
    const double2* V0 = VAL(K);
    const double* W0 = WV(K);
    // ---- plane z + 1, own rows: the z faces, and next step's own values
    double2 nxt[YB];
    double wnx[YB];
    int lnx[YB];
    double crc[YB], crp[YB];
#pragma unroll
    for (int i = 0; i < YB; ++i) {
      const int r = ty0 + i + 1;
      nxt[i] = VAL(K1)[qi(r)];
      lnx[i] = LAB(K1)[li(r)];
      wnx[i] = OC ? WV(K1)[di(r)] : 0.0;
      double fc, fp;
      face(lcur[i], cur[i], wcur[i], lnx[i], nxt[i], wnx[i], fc, fp);
      rc[i] += fc;
      rp[i] += fp;
      crc[i] = -fc;
      crp[i] = -fp;
    }
    // ---- y faces: between own rows, then to the rows outside (tile halo / other warps)
#pragma unroll
    for (int i = 0; i + 1 < YB; ++i) {
      double fc, fp;
      face(lcur[i], cur[i], wcur[i], lcur[i + 1], cur[i + 1], wcur[i + 1], fc, fp);
      rc[i] += fc;
      rp[i] += fp;
      rc[i + 1] -= fc;
      rp[i + 1] -= fp;
    }
    {   // y faces to the rows outside this thread (tile halo / other warps)
      const int rlo = ty0, rhi = ty0 + YB + 1;   // smem rows of those neighbours
      double fc, fp;
      face(lcur[0], cur[0], wcur[0], L0[li(rlo)], V0[qi(rlo)], OC ? W0[di(rlo)] : 0.0, fc, fp);
      rc[0] += fc;
      rp[0] += fp;
      face(lcur[YB - 1], cur[YB - 1], wcur[YB - 1], L0[li(rhi)], V0[qi(rhi)], OC ? W0[di(rhi)] : 0.0, fc, fp);
      rc[YB - 1] += fc;
      rp[YB - 1] += fp;
    }
    // ---- x faces: (x, x+1) here, its negative handed to lane x+1
#pragma unroll
    for (int i = 0; i < YB; ++i) {
      const int r = ty0 + i + 1;
      double2 vb;
      vb.x = __shfl_down_sync(0xffffffffu, cur[i].x, 1);
      vb.y = __shfl_down_sync(0xffffffffu, cur[i].y, 1);
      double wb = OC ? __shfl_down_sync(0xffffffffu, wcur[i], 1) : 0.0;
      int lb = __shfl_down_sync(0xffffffffu, lcur[i], 1);
      if (lane == VX - 1) {   // right tile halo
        vb = V0[qi(r) + 1];
        lb = L0[li(r) + 1];
        wb = OC ? W0[di(r) + 1] : 0.0;
      }
      double fc, fp;
      face(lcur[i], cur[i], wcur[i], lb, vb, wb, fc, fp);
      rc[i] += fc;
      rp[i] += fp;
      const double gc = __shfl_up_sync(0xffffffffu, fc, 1), gp = __shfl_up_sync(0xffffffffu, fp, 1);
      if (lane > 0) {
        rc[i] -= gc;
        rp[i] -= gp;
      } else {   // left tile halo: this lane evaluates the face itself
        face(lcur[i], cur[i], wcur[i], L0[li(r) - 1], V0[qi(r) - 1], OC ? W0[di(r) - 1] : 0.0, fc, fp);
        rc[i] += fc;
        rp[i] += fp;
      }
    }
    // ---- interface faces (the row's own alpha, beta, gamma per masked direction; the
    // neighbour values of plane z come from the staged tile) and rows out
#pragma unroll
    for (int i = 0; i < YB; ++i) {
      double si = 0.0;
      const unsigned mask = ((unsigned)lcur[i] >> 3) & 63u;
      if (mask) {
        const int r = ty0 + i + 1;
        const int gs = (int)((unsigned)lcur[i] >> 9), loc = gs - tp_start[K];
        const double* c = loc + __popc(mask) <= T_SLOTCAP
                              ? reinterpret_cast<const double*>(ring + K * L::SLOT + L::SLT) + 4 * loc
                              : F.cslot + 4LL * gs;
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          if (mask & (1u << d)) {
            const double2 vb = d == 4 ? prv[i] : d == 5 ? nxt[i]
                             : V0[d == 0 ? qi(r) - 1 : d == 1 ? qi(r) + 1 : d == 2 ? qi(r - 1) : qi(r + 1)];
            const double2 ab = *reinterpret_cast<const double2*>(c);
            si += ab.x * cur[i].x + ab.y * vb.x + c[2] * (cur[i].y - vb.y);
            c += 4;
          }
        }
      }
      const int y = y0 + ty0 + i;
      if (x < nx && y < ny) {
        const int a = lcur[i] & 7;
        const long long v = (long long)z * nxy + (long long)y * nx + x;
        const bool in_row = !(z == nz - 1 && a == TCC);
        double c_ = rc[i], p_ = rp[i];
        if (!in_row) {
          c_ = p_ = 0.0;
        } else {
          const bool crow = a == TGR || a == TEL;
          if (a == TEL) c_ = (flags & 2) ? fma(1.0 - tp, si, c_) : fma(tp, p_, c_) + si;
          else if (crow) c_ += si;
          p_ += si;
          if ((flags & 1) && crow) c_ = fma(cur[i].x, inv_dt, c_);
          if (flags & 8) c_ = 0.0;
        }
        out2[v] = make_double2(c_, p_);
        if (F.dot_a) {
          const double2 da = F.dot_a[v];
          dacc1 += c_ * da.x + p_ * da.y;
          dacc2 += c_ * c_ + p_ * p_;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * K);   // this warp is done with plane z
#pragma unroll
    for (int i = 0; i < YB; ++i) {
      prv[i] = cur[i];
      cur[i] = nxt[i];
      wcur[i] = wnx[i];
      lcur[i] = lnx[i];
      rc[i] = crc[i];
      rp[i] = crp[i];
    }
  };
  for (int jb = 0; jb < nplane; jb += T_S) {
    const unsigned ph = (jb / T_S) & 1;
    static_for<T_S>([&](auto kc) {
      constexpr int K = decltype(kc)::value;
      if (jb + K < nplane) step(jb + K, kc, K + 1 == T_S ? ph ^ 1 : ph);
    });
  }
  if (F.dot_a) {
    __shared__ double dsh[2][NW];
    for (int o = 16; o > 0; o >>= 1) {
      dacc1 += __shfl_down_sync(0xffffffffu, dacc1, o);
      dacc2 += __shfl_down_sync(0xffffffffu, dacc2, o);
    }
    if (lane == 0) {
      dsh[0][warp] = dacc1;
      dsh[1][warp] = dacc2;
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(NW * VX) : "memory");
    if (tid == 0) {
      double a1 = 0.0, a2 = 0.0;
      for (int k = 0; k < NW; ++k) {
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

// J v through the register-blocked kernel; false if the grid / pointers do not allow
// tensor-map tiles (the caller falls back)
template <int YB>
inline bool jv_launch_y(TmaCache& cache, const DevParams& P, const FineArgs& F, const int32_t* labt,
                        const double2* V, double inv_dt, int flags, double2* out2, int n_sm, cudaStream_t s) {
  using L = TmaLayout<SM_FULL, EP_STORE>;
  if (!tma_grid_ok(P) || !labt) return false;
  TmaMaps M;
  std::memset(&M, 0, sizeof(M));
  const CUtensorMap* m = tma_map(cache, labt, 0, P.nx, P.ny, P.nz);
  if (!m) return false;
  M.lab = *m;
  if (!(m = tma_map(cache, V, 1, P.nx, P.ny, P.nz))) return false;
  M.val = *m;
  const bool oc = flags & 4;
  if (oc) {
    if (!(m = tma_map(cache, F.w, 2, P.nx, P.ny, P.nz))) return false;
    M.aux = *m;
  }
  const size_t smem = (size_t)T_S * L::SLOT + 128;
  const int bx = (P.nx + VX - 1) / VX, by = (P.ny + VY - 1) / VY;
  auto go = [&](auto onec) {
    constexpr bool OC = decltype(onec)::value;
    auto kern = k_jv_y<YB, OC>;
    static int per_sm = 0;
    if (!per_sm) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, YLayout<YB>::THREADS, smem);
      if (per_sm < 1) per_sm = 1;
    }
    const int bz = pick_bz(bx, by, P.nz, per_sm, n_sm);
    const int zc = (P.nz + bz - 1) / bz;
    const dim3 grid(bx, by, (P.nz + zc - 1) / zc);
    if (F.dot_nblk) *F.dot_nblk = (int)(grid.x * grid.y * grid.z);
    launch(kern, grid, dim3(VX, YLayout<YB>::THREADS / VX, 1), smem, s, P, M, F, labt, V, inv_dt, flags,
           out2, zc);
  };
  if (oc) go(std::true_type{});
  else go(std::false_type{});
  return true;
}

}  // namespace hc
