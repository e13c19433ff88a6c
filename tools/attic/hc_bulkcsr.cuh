// Bulk-fed CSR gather kernels for the multigrid's coarse levels and transfers.
//
// The CSR sweeps / restrictions / prolongations of the preconditioner were latency-bound
// (ncu: long-scoreboard stalls, ~0.5 eligible warps per scheduler, DRAM ~30 % busy):
// every row is a chain of dependent loads  row pointer -> column index / value -> x[col].
// Here the rows are cut (once per sparsity pattern, on the host) into chunks of at most
// BK_CAP nonzeros; a producer warp streams each chunk's row-pointer, column-index and
// value slices — and, for the smoothing sweeps, its right-hand side and D^-1 slices —
// into a BK_ST-deep shared-memory ring with cp.async.bulk (TMA bulk copies, mbarrier
// completion), so the only dependent global loads left are the gathers x[col], which
// hit L2 (the level vectors are L2-resident).  CTAs are persistent (a few per SM) and
// loop over the chunks.
//
// KIND 0/1/2: the smoothing sweep of k_csr_x with input mode XM = KIND
//             (y = xin + w D^-1 (b - A xin), or with resid y = b - A xin);
// KIND 3:     y[i] = sum_k v[k] g[col[k]]            (restriction P^T r);
// KIND 4:     y[i] += alpha sum_k v[k] g[col[k]]     (prolongation, rows without entries untouched).
#pragma once

#include "hc_tma.cuh"

namespace hc {

constexpr int BK_CAP = 2048;    // nonzeros per chunk
constexpr int BK_ROWS = 256;    // rows per chunk
constexpr int BK_ST = 3;        // ring depth
constexpr int BK_WARPS = 8;     // consumer warps per CTA

struct BulkArgs {
  int n_chunk;
  const int2* chunk;      // [n_chunk + 1]: (first row, first nonzero) of every chunk
  const int32_t* rp;
  const int32_t* ci;
  const void* v;          // float or double values
  double w, alpha;
  const double* b;        // sweeps: right-hand side;  KIND 3/4: unused
  const double* x;        // sweeps: current iterate (XM 0/2)
  const double* dinv;
  const int32_t* parent;  // XM 2
  const double* xc;       // XM 2: coarse correction
  const double* g;        // KIND 3/4: gathered vector
  double* y;
  double* x0;             // sweeps with resid: also store the input iterate
  int resid;
};

template <class VT>
struct BkLayout {
  static constexpr int RP = 0;                                                     // int32 [BK_ROWS + 8]
  static constexpr int CI = ((BK_ROWS + 8) * 4 + 127) / 128 * 128;                // int32 [BK_CAP + 4]
  static constexpr int VV = CI + ((BK_CAP + 4) * 4 + 127) / 128 * 128;             // VT [BK_CAP + 4]
  static constexpr int BB = VV + ((BK_CAP + 4) * (int)sizeof(VT) + 127) / 128 * 128;   // double [BK_ROWS + 2]
  static constexpr int DD = BB + ((BK_ROWS + 2) * 8 + 127) / 128 * 128;            // double [BK_ROWS + 2]
  static constexpr int STAGE = DD + ((BK_ROWS + 2) * 8 + 127) / 128 * 128;
  static constexpr int THREADS = 32 * (BK_WARPS + 1);
};

template <int VS, class VT, int KIND>
__global__ void __launch_bounds__(BkLayout<VT>::THREADS)
k_csr_bulk(BulkArgs A) {
  using L = BkLayout<VT>;
  constexpr bool SWEEP = KIND <= 2;
  extern __shared__ __align__(16) unsigned char bk_dyn[];
  unsigned char* ring = bk_dyn + ((128 - ((unsigned)__cvta_generic_to_shared(bk_dyn) & 127)) & 127);
  __shared__ __align__(8) unsigned long long full[BK_ST], empty[BK_ST];
  __shared__ int hdr[BK_ST][5];   // r0, r1, ra (rp slice start), ka (nonzero slice start), rb (row-vector slice start)
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(full);
  const unsigned empty0 = (unsigned)__cvta_generic_to_shared(empty);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < BK_ST; ++k) {
      mbar_init(full0 + 8 * k, 1);
      mbar_init(empty0 + 8 * k, BK_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();

  if (warp == BK_WARPS) {   // ------------------------------- producer warp
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(ring);
    // chunk descriptors of the next 32 own chunks, one per lane (no dependent round trip
    // per chunk on the issue path)
    int2 lo_l = make_int2(0, 0), hi_l = make_int2(0, 0);
    auto fetch = [&](int c0) {
      const int c = c0 + lane * (int)gridDim.x;
      if (c < A.n_chunk) {
        lo_l = A.chunk[c];
        hi_l = A.chunk[c + 1];
      }
    };
    int it = 0;
    for (int cb = blockIdx.x; cb < A.n_chunk; cb += 32 * gridDim.x) {
      fetch(cb);
      for (int q = 0; q < 32; ++q, ++it) {
        const int c = cb + q * (int)gridDim.x;
        if (c >= A.n_chunk) break;
        const int r0 = __shfl_sync(0xffffffffu, lo_l.x, q), k0 = __shfl_sync(0xffffffffu, lo_l.y, q);
        const int r1 = __shfl_sync(0xffffffffu, hi_l.x, q), k1 = __shfl_sync(0xffffffffu, hi_l.y, q);
        if (lane == 0) {
          const int s = it % BK_ST;
          if (it >= BK_ST) mbar_wait(empty0 + 8 * s, ((it / BK_ST) - 1) & 1);
          const int ra = r0 & ~3, ka = k0 & ~3, rb = r0 & ~1;
          hdr[s][0] = r0; hdr[s][1] = r1; hdr[s][2] = ra; hdr[s][3] = ka; hdr[s][4] = rb;
          const unsigned brp = ((r1 + 1 - ra) * 4 + 15) & ~15u;
          const unsigned bci = ((k1 - ka) * 4 + 15) & ~15u;
          const unsigned bv = ((k1 - ka) * (int)sizeof(VT) + 15) & ~15u;
          const unsigned bb = SWEEP ? (((r1 - rb) * 8 + 15) & ~15u) : 0u;
          const unsigned b = full0 + 8 * s, st = sbase + s * L::STAGE;
          mbar_expect_tx(b, brp + bci + bv + 2 * bb);
          bulk_load(st + L::RP, A.rp + ra, brp, b);
          if (bci) {
            bulk_load(st + L::CI, A.ci + ka, bci, b);
            bulk_load(st + L::VV, reinterpret_cast<const VT*>(A.v) + ka, bv, b);
          }
          if (SWEEP && bb) {
            bulk_load(st + L::BB, A.b + rb, bb, b);
            bulk_load(st + L::DD, A.dinv + rb, bb, b);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumer warps
  constexpr int G = BK_WARPS * 32 / VS;               // row groups
  const int grp = (warp * 32 + lane) / VS, lg = lane % VS;
  auto xin = [&](int j, const double* bs, const double* ds, int rb) -> double {
    if (KIND == 0) return __ldg(A.x + j);
    if (KIND == 1) return A.w * ds[j - rb] * bs[j - rb];   // own row only (staged)
    return __ldg(A.x + j) + A.alpha * __ldg(A.xc + __ldg(A.parent + j));
  };
  auto gat = [&](int j) -> double {
    if (KIND == 0) return __ldg(A.x + j);
    if (KIND == 1) return A.w * __ldg(A.dinv + j) * __ldg(A.b + j);
    if (KIND == 2) return __ldg(A.x + j) + A.alpha * __ldg(A.xc + __ldg(A.parent + j));
    return __ldg(A.g + j);
  };
  int it = 0;
  for (int c = blockIdx.x; c < A.n_chunk; c += gridDim.x, ++it) {
    const int s = it % BK_ST;
    mbar_wait(full0 + 8 * s, (it / BK_ST) & 1);
    const unsigned char* S = ring + s * L::STAGE;
    const int r0 = hdr[s][0], r1 = hdr[s][1], ra = hdr[s][2], ka = hdr[s][3], rb = hdr[s][4];
    const int* rps = reinterpret_cast<const int*>(S + L::RP);
    const int* cis = reinterpret_cast<const int*>(S + L::CI);
    const VT* vs = reinterpret_cast<const VT*>(S + L::VV);
    const double* bs = reinterpret_cast<const double*>(S + L::BB);
    const double* ds = reinterpret_cast<const double*>(S + L::DD);
    for (int rbase = r0; rbase < r1; rbase += G) {
      const int r = rbase + grp;
      const bool ok = r < r1;
      double sum = 0.0;
      int kb = 0, ke = 0;
      if (ok) {
        kb = rps[r - ra] - ka;
        ke = rps[r + 1 - ra] - ka;
        int k = kb + lg;
        for (; k + 3 * VS < ke; k += 4 * VS) {
          const int c0 = cis[k], c1 = cis[k + VS], c2 = cis[k + 2 * VS], c3 = cis[k + 3 * VS];
          const double a0 = (double)vs[k], a1 = (double)vs[k + VS], a2 = (double)vs[k + 2 * VS],
                       a3 = (double)vs[k + 3 * VS];
          const double x0 = gat(c0), x1 = gat(c1), x2 = gat(c2), x3 = gat(c3);
          sum += a0 * x0;
          sum += a1 * x1;
          sum += a2 * x2;
          sum += a3 * x3;
        }
        for (; k < ke; k += VS) sum += (double)vs[k] * gat(cis[k]);
      }
      if (VS > 1) {
#pragma unroll
        for (int o = VS / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, VS);
      }
      if (ok && lg == 0) {
        if constexpr (SWEEP) {
          const double xi = xin(r, bs, ds, rb);
          const double bi = bs[r - rb];
          A.y[r] = A.resid ? bi - sum : xi + A.w * ds[r - rb] * (bi - sum);
          if (A.x0) A.x0[r] = xi;
        } else if constexpr (KIND == 3) {
          A.y[r] = sum;
        } else {
          if (ke > kb) A.y[r] += A.alpha * sum;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s);
  }
}

// Chunk descriptors (host): rows cut so that no chunk holds more than BK_CAP nonzeros or
// BK_ROWS rows.  Returns false if a single row exceeds BK_CAP (the caller keeps the
// per-row kernels for that matrix).
inline bool bulk_chunks(const std::vector<int32_t>& rp, std::vector<int2>& out) {
  out.clear();
  const int n = (int)rp.size() - 1;
  int r = 0;
  while (r < n) {
    out.push_back(make_int2(r, rp[r]));
    int e = r;
    while (e < n && e - r < BK_ROWS && rp[e + 1] - rp[r] <= BK_CAP) ++e;
    if (e == r) return false;   // row r alone exceeds the chunk capacity
    r = e;
  }
  out.push_back(make_int2(n, n ? rp[n] : 0));
  return true;
}

}  // namespace hc
