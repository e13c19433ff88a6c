// POD snapshot Gram matrix G = S^T diag(w) S (method of snapshots, SPEC mor.pod),
// the only dense contraction of the path.  S is n_dof x n_snap fp64, column-major or
// row-major (snapshots contiguous per DOF: a DOF chunk of every snapshot is one block,
// so concurrent CTAs share pages and L2 lines; no transpose copy is needed).
//
// FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).  Each CTA owns one 64x64 tile of
// the upper triangle of G (G is symmetric: 28 of 49 tiles for 400 snapshots) and
// one slice of the DOF dimension (split-K).  The DOF chunks of both operand panels
// and of the weights stream through a 3-stage cp.async ring in shared memory, so
// HBM/L2 traffic overlaps the DMMA work; 4 warps each own a 32x32 sub-tile (16 DMMA
// per k-step from 8 fragment loads).  Slices are reduced in a fixed order and the
// triangle mirrored, so the result is deterministic and exactly symmetric.
#include <algorithm>

#include "hc_internal.cuh"

namespace hc {

namespace {
constexpr int BT = 64;      // tile of G
constexpr int KC = 32;      // DOF chunk per stage
constexpr int ST = 3;       // pipeline stages
constexpr int LD = KC + 2;  // padded row of a staged panel
constexpr int NT = 128;     // 4 warps: 2 x 2 sub-tiles of 32 x 32

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 8-byte async copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp8(void* smem, const void* gmem, int src_bytes) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// part[z][j * n + i] = sum_{k in slice z} S[k][i] w[k] S[k][j]   for the tile pair (ti <= tj)
template <bool ROWS>
__global__ void __launch_bounds__(NT) k_gram(const double* __restrict__ S, const double* __restrict__ w,
                                             long long n_dof, int n, int tiles, long long k_per,
                                             double* __restrict__ part) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                        // [ST][BT][LD]
  double* Bs = As + ST * BT * LD;           // [ST][BT][LD]
  double* Ws = Bs + ST * BT * LD;           // [ST][KC]
  // upper-triangle tile pair from the linear block index
  int p = blockIdx.x, ti = 0;
  while (p >= tiles - ti) { p -= tiles - ti; ++ti; }
  const int tj = ti + p;
  const int i0 = ti * BT, j0 = tj * BT, z = blockIdx.y;
  const long long k_begin = (long long)z * k_per;
  const long long k_end = min(n_dof, k_begin + k_per);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int g = lane >> 2, tq = lane & 3;
  const double* wsrc = w;
  auto stage = [&](long long k0, int s) {
    // 64 columns x 32 DOFs per panel: 2048 elements per panel, 16 per thread
    for (int e = tid; e < BT * KC; e += NT) {
      // column-major S: consecutive threads walk k (a column's 256 B); row-major S
      // (snapshots contiguous per DOF): consecutive threads walk the 64 snapshots of one
      // DOF row, and a whole 32-DOF chunk of all snapshots is one contiguous block
      const int col = ROWS ? e % BT : e / KC, kk = ROWS ? e / BT : e - col * KC;
      const long long k = k0 + kk;
      const int gi = i0 + col, gj = j0 + col;
      const bool kin = k < k_end;
      const long long kk0 = kin ? k : 0;
      const double* ai = ROWS ? S + kk0 * n + min(gi, n - 1) : S + (long long)min(gi, n - 1) * n_dof + kk0;
      const double* bj = ROWS ? S + kk0 * n + min(gj, n - 1) : S + (long long)min(gj, n - 1) * n_dof + kk0;
      cp8(As + (s * BT + col) * LD + kk, ai, (kin && gi < n) ? 8 : 0);
      cp8(Bs + (s * BT + col) * LD + kk, bj, (kin && gj < n) ? 8 : 0);
    }
    if (tid < KC) {
      const long long k = k0 + tid;
      const bool kin = k < k_end;
      if (wsrc) cp8(Ws + s * KC + tid, wsrc + (kin ? k : 0), kin ? 8 : 0);
      else Ws[s * KC + tid] = kin ? 1.0 : 0.0;
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const long long nchunks = (k_end - k_begin + KC - 1) / KC;
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) {
    if (s < nchunks) stage(k_begin + (long long)s * KC, s);
    cp_commit();
  }
  for (long long c = 0; c < nchunks; ++c) {
    cp_wait<ST - 2>();
    __syncthreads();
    const long long cn = c + ST - 1;
    if (cn < nchunks) stage(k_begin + cn * KC, (int)(cn % ST));
    cp_commit();
    const int s = (int)(c % ST);
    const double* A = As + s * BT * LD;
    const double* B = Bs + s * BT * LD;
    const double* W = Ws + s * KC;
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      const double wk = W[ks + tq];
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = A[(wr * 32 + a * 8 + g) * LD + ks + tq] * wk;
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = B[(wc * 32 + b * 8 + g) * LD + ks + tq];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_wait<0>();
  double* out = part + (long long)z * n * n;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + wr * 32 + a * 8 + g;
      const int j = j0 + wc * 32 + b * 8 + tq * 2;
      if (i < n && j < n) out[(long long)j * n + i] = acc[a][b][0];
      if (i < n && j + 1 < n) out[(long long)(j + 1) * n + i] = acc[a][b][1];
    }
}

// G[j][i] = G[i][j] = sum_z part[z] over the upper triangle (fixed order)
__global__ void k_reduce_sym(int n, int nz, int tiles, const double* __restrict__ part,
                             double* __restrict__ G) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nn = (long long)n * n;
  if (e >= nn) return;
  const int j = (int)(e / n), i = (int)(e % n);
  // the tile pair (ti <= tj) that computed this entry
  const int ti = i / BT, tj = j / BT;
  const bool upper = ti <= tj;
  const long long src = upper ? e : (long long)i * n + j;   // mirrored entry
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += part[(long long)z * nn + src];
  G[e] = s;
  (void)tiles;
}
}  // namespace

void pod_gram(const double* S, const double* w, long long n_dof, long long n_snap, double* G,
              cudaStream_t s, bool rows) {
  if (n_snap == 0) return;
  const int n = (int)n_snap;
  const int tiles = (n + BT - 1) / BT;
  const int pairs = tiles * (tiles + 1) / 2;
  int sms = 148, dev = 0;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = (size_t)(2 * ST * BT * LD + ST * KC) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    HC_CUDA(cudaFuncSetAttribute(k_gram<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HC_CUDA(cudaFuncSetAttribute(k_gram<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int per_sm = 1;
  HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gram<false>, NT, smem));
  const long long want = std::max<long long>(1, ((long long)std::max(per_sm, 1) * sms + pairs - 1) / pairs);
  long long k_per = (n_dof + want - 1) / want;
  k_per = std::max<long long>(KC, ((k_per + KC - 1) / KC) * KC);
  const int nz = (int)std::max<long long>(1, (n_dof + k_per - 1) / k_per);
  DBuf<double> part((size_t)nz * n * n);
  HC_CUDA(cudaMemsetAsync(part.p, 0, part.n * sizeof(double), s));
  if (rows) k_gram<true><<<dim3(pairs, nz), NT, smem, s>>>(S, w, n_dof, n, tiles, k_per, part.p);
  else k_gram<false><<<dim3(pairs, nz), NT, smem, s>>>(S, w, n_dof, n, tiles, k_per, part.p);
  HC_COUNT();
  HC_CHECK_LAUNCH();
  const long long nn = (long long)n * n;
  k_reduce_sym<<<(int)((nn + 255) / 256), 256, 0, s>>>(n, nz, tiles, part.p, G); HC_COUNT();
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hc
