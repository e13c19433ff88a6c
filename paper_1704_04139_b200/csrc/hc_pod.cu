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
#include <cstdint>

#include "hc_internal.cuh"

namespace hc {

namespace {
constexpr int BT = 64;      // tile of G
constexpr int KC = 16;      // K chunk per stage (16: 55 KB of ring per CTA, 4 CTAs / 16 warps per SM)
constexpr int ST = 3;       // pipeline stages
constexpr int LD = KC + 2;  // padded row of a staged panel, [col][k] layout (k contiguous in memory or generic strides)
constexpr int LDI = BT + 4; // padded row of a staged panel, [k][col] layout (tile index contiguous in memory):
                            // 16-byte copies of column pairs; LDI mod 16 == 4 keeps the fragment loads conflict-free
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
// 16-byte async copy (two doubles); src_bytes 8 copies one and zero-fills the other, 0 zero-fills both
__device__ __forceinline__ void cp16(void* smem, const void* gmem, int src_bytes) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Generic FP64 tensor-core contraction  C[i][j] = sum_k w[k] A(k, i) B(k, j)  with strided
// operands A(k, i) = A[k sa_k + i sa_i], B(k, j) = B[k sb_k + j sb_j]:
//   * the POD Gram S^T W S (sym: upper-triangle tile pairs only, A == B, mirrored),
//   * tall-times-small projections S (U / sigma), V R^-1, W[:, :l] X (i over DOFs, k short),
//   * long-inner-dimension products B^T W (i, j short, k over DOFs; split-K).
// One CTA per 64 x 64 tile of C (and K slice); both operand panels and the weights stream
// through a 3-stage cp.async ring, 4 warps each own a 32 x 32 sub-tile (16 DMMA
// m8n8k4 per k-step from 8 fragment loads).  Split-K partials are reduced in a fixed order.
struct GemmDesc {
  const double* A;
  long long sa_k, sa_i;
  const double* B;
  long long sb_k, sb_j;
  const double* w;       // optional weights over k
  long long K;
  int M, N, tiles_i, tiles_j, sym;
  long long k_per;
  double* out;           // nz == 1: C (row-major, ldc);  else partials [z][M][N]
  long long ldc;
};

// AI / BJ: the tile index of A / B is the contiguous one in memory (stride 1, even k stride,
// 16-byte aligned base): that panel is staged [k][col] with 16-byte copies of column pairs — a
// thread keeps its column pair and walks k, so the copy loop is a pointer increment per copy
// instead of the generic path's per-element index arithmetic (which issued more instructions
// than the DMMA loop itself).
constexpr int PANEL = ST * (BT * LD > KC * LDI ? BT * LD : KC * LDI);   // doubles per operand ring

template <bool AI, bool BJ>
__global__ void __launch_bounds__(NT) k_dgemm(GemmDesc D) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                        // [ST][BT][LD] or [ST][KC][LDI]
  double* Bs = As + PANEL;
  double* Ws = Bs + PANEL;                  // [ST][KC]
  int ti, tj;
  if (D.sym) {   // upper-triangle tile pair from the linear block index
    int p = blockIdx.x;
    ti = 0;
    while (p >= D.tiles_i - ti) { p -= D.tiles_i - ti; ++ti; }
    tj = ti + p;
  } else {
    ti = blockIdx.x / D.tiles_j;
    tj = blockIdx.x - ti * D.tiles_j;
  }
  const int i0 = ti * BT, j0 = tj * BT, z = blockIdx.y;
  const long long k_begin = (long long)z * D.k_per;
  const long long k_end = min(D.K, k_begin + D.k_per);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;
  const int g = lane >> 2, tq = lane & 3;
  // staging order: walk whichever index is contiguous in memory
  const bool a_icont = D.sa_i == 1, b_jcont = D.sb_j == 1;
  // [k][col] staging of a tile-contiguous panel: thread = (column pair, k mod 4)
  auto stage_pairs = [&](const double* base, long long sk, int t0, int lim, double* dst, long long k0, int s) {
    const int cp = tid & 31, kq = tid >> 5;
    const int gt = t0 + 2 * cp;
    const int full = gt + 1 < lim ? 16 : (gt < lim ? 8 : 0);
    const double* src = base + (k0 + kq) * sk + gt;
    double* d = dst + (s * KC + kq) * LDI + 2 * cp;
#pragma unroll
    for (int it = 0; it < KC / 4; ++it) {
      const int bytes = k0 + kq + 4 * it < k_end ? full : 0;
      cp16(d, bytes ? src : base, bytes);
      src += 4 * sk;
      d += 4 * LDI;
    }
  };
  auto stage = [&](long long k0, int s) {
    if constexpr (AI) stage_pairs(D.A, D.sa_k, i0, D.M, As, k0, s);
    if constexpr (BJ) stage_pairs(D.B, D.sb_k, j0, D.N, Bs, k0, s);
    if constexpr (!AI || !BJ) {
      for (int e = tid; e < BT * KC; e += NT) {
        if constexpr (!AI) {
          const int col = a_icont ? e % BT : e / KC, kk = a_icont ? e / BT : e - (e / KC) * KC;
          const long long k = k0 + kk;
          const int gi = i0 + col;
          const bool ok = k < k_end && gi < D.M;
          const double* src = D.A + (ok ? k * D.sa_k + (long long)gi * D.sa_i : 0);
          cp8(As + (s * BT + col) * LD + kk, src, ok ? 8 : 0);
        }
        if constexpr (!BJ) {
          const int col = b_jcont ? e % BT : e / KC, kk = b_jcont ? e / BT : e - (e / KC) * KC;
          const long long k = k0 + kk;
          const int gj = j0 + col;
          const bool ok = k < k_end && gj < D.N;
          const double* src = D.B + (ok ? k * D.sb_k + (long long)gj * D.sb_j : 0);
          cp8(Bs + (s * BT + col) * LD + kk, src, ok ? 8 : 0);
        }
      }
    }
    if (tid < KC) {
      const long long k = k0 + tid;
      const bool kin = k < k_end;
      if (D.w) cp8(Ws + s * KC + tid, D.w + (kin ? k : 0), kin ? 8 : 0);
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
    const double* A = As + s * (AI ? KC * LDI : BT * LD);
    const double* B = Bs + s * (BJ ? KC * LDI : BT * LD);
    const double* W = Ws + s * KC;
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      const double wk = W[ks + tq];
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        af[a] = (AI ? A[(ks + tq) * LDI + wr * 32 + a * 8 + g] : A[(wr * 32 + a * 8 + g) * LD + ks + tq]) * wk;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        bf[b] = BJ ? B[(ks + tq) * LDI + wc * 32 + b * 8 + g] : B[(wc * 32 + b * 8 + g) * LD + ks + tq];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_wait<0>();
  const bool direct = gridDim.y == 1;
  double* out = direct ? D.out : D.out + (long long)z * D.M * D.N;
  const long long ld = direct ? D.ldc : D.N;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + wr * 32 + a * 8 + g;
      const int j = j0 + wc * 32 + b * 8 + tq * 2;
      if (i < D.M && j < D.N) out[(long long)i * ld + j] = acc[a][b][0];
      if (i < D.M && j + 1 < D.N) out[(long long)i * ld + j + 1] = acc[a][b][1];
    }
}

// FP64 tensor-core throughput probe: every warp issues `iters` x 16 independent DMMA
// m8n8k4 on register operands (no memory traffic); 2 * 8 * 8 * 4 flops each
__global__ void __launch_bounds__(NT) k_dmma_peak(long long iters, double* sink) {
  double acc[16][2];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q][0] = acc[q][1] = 0.0;
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 16; ++q) dmma_8x8x4(acc[q][0], acc[q][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += acc[q][0] + acc[q][1];
  if (s == 12345.0) sink[0] = s;
}

// C[i][j] = sum_z part[z][i][j] (fixed order); sym: the lower triangle mirrors the upper
__global__ void k_reduce_parts(int M, int N, int nz, int sym, const double* __restrict__ part,
                               double* __restrict__ C, long long ldc) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long mn = (long long)M * N;
  if (e >= mn) return;
  const int i = (int)(e / N), j = (int)(e % N);
  const long long src = (sym && i / BT > j / BT) ? (long long)j * N + i : e;   // tile computed as (tj, ti)
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += part[(long long)z * mn + src];
  C[(long long)i * ldc + j] = s;
}
}  // namespace

// C (M x N, row-major, ldc) = sum_k w[k] A(k, i) B(k, j) on the FP64 tensor cores
void dgemm_tc(const double* A, long long sa_k, long long sa_i, const double* B, long long sb_k, long long sb_j,
              const double* w, long long K, int M, int N, double* C, long long ldc, bool sym, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    for (int i = 0; i < M; ++i) HC_CUDA(cudaMemsetAsync(C + (long long)i * ldc, 0, N * sizeof(double), s));
    return;
  }
  const int tiles_i = (M + BT - 1) / BT, tiles_j = (N + BT - 1) / BT;
  const long long pairs = sym ? (long long)tiles_i * (tiles_i + 1) / 2 : (long long)tiles_i * tiles_j;
  int sms = 148, dev = 0;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = (size_t)(2 * PANEL + ST * KC) * sizeof(double);
  // tile-contiguous operands with 16-byte aligned column pairs take the [k][col] staging
  auto pairable = [](const double* p, long long s_k, long long s_t) {
    return s_t == 1 && s_k % 2 == 0 && reinterpret_cast<uintptr_t>(p) % 16 == 0;
  };
  const bool ai = pairable(A, sa_k, sa_i), bj = pairable(B, sb_k, sb_j);
  void (*kern)(GemmDesc) = ai ? (bj ? k_dgemm<true, true> : k_dgemm<true, false>)
                              : (bj ? k_dgemm<false, true> : k_dgemm<false, false>);
  static int per_sm_v[4] = {0, 0, 0, 0};
  int& per_sm = per_sm_v[(ai ? 2 : 0) | (bj ? 1 : 0)];
  if (!per_sm) {
    HC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
    per_sm = std::max(per_sm, 1);
  }
  // split K only when the tiles alone cannot fill the GPU
  const long long want = std::max<long long>(1, ((long long)per_sm * sms + pairs - 1) / pairs);
  long long k_per = (K + want - 1) / want;
  k_per = std::max<long long>(KC, ((k_per + KC - 1) / KC) * KC);
  const int nz = (int)std::max<long long>(1, (K + k_per - 1) / k_per);
  GemmDesc D{A, sa_k, sa_i, B, sb_k, sb_j, w, K, M, N, tiles_i, tiles_j, sym ? 1 : 0, k_per, C, ldc};
  // split-K partials: a per-thread buffer that only grows (a cudaMalloc / cudaFree pair per call
  // cost up to 10 ms of the 20 ms Gram when the allocator had to map fresh memory); this function
  // synchronises the stream before it returns whenever the buffer was used, so reuse is safe
  static thread_local DBuf<double> part;
  const size_t need = (nz > 1 || sym) ? (size_t)nz * M * N : 0;
  if (need) {
    if (part.n < need) part.alloc(need);
    if (sym) HC_CUDA(cudaMemsetAsync(part.p, 0, need * sizeof(double), s));
    D.out = part.p;
  }
  if (pairs > 0x7fffffffLL) throw Error(HC_ERR_ARGUMENT, "contraction too large");
  // nz == 1 with sym still goes through the partial buffer (the mirror pass)
  kern<<<dim3((unsigned)pairs, nz), NT, smem, s>>>(D);
  HC_COUNT();
  HC_CHECK_LAUNCH();
  if (need) {
    const long long mn = (long long)M * N;
    k_reduce_parts<<<(int)((mn + 255) / 256), 256, 0, s>>>(M, N, nz, sym ? 1 : 0, part.p, C, ldc); HC_COUNT();
    HC_CHECK_LAUNCH();
    HC_CUDA(cudaStreamSynchronize(s));   // the partial buffer is reused by the next call
  }
}

// measured FP64 DMMA throughput (TFLOP/s) of the whole GPU
double dmma_peak_tflops(cudaStream_t s) {
  int sms = 148, dev = 0;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DBuf<double> sink(1);
  const long long iters = 20000;
  const int grid = sms * 8;
  k_dmma_peak<<<grid, NT, 0, s>>>(1000, sink.p);   // warm
  HC_COUNT();
  cudaEvent_t e0, e1;
  HC_CUDA(cudaEventCreate(&e0));
  HC_CUDA(cudaEventCreate(&e1));
  HC_CUDA(cudaEventRecord(e0, s));
  k_dmma_peak<<<grid, NT, 0, s>>>(iters, sink.p);
  HC_COUNT();
  HC_CUDA(cudaEventRecord(e1, s));
  HC_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  HC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = (double)grid * (NT / 32) * iters * 16 * 2.0 * 8 * 8 * 4;
  return flops / (ms * 1e-3) / 1e12;
}

void pod_gram(const double* S, const double* w, long long n_dof, long long n_snap, double* G,
              cudaStream_t s, bool rows) {
  if (n_snap == 0) return;
  // A(k, i) = S[k][i]: row-major S (snapshots contiguous per DOF) or column-major
  if (rows) dgemm_tc(S, n_snap, 1, S, n_snap, 1, w, n_dof, (int)n_snap, (int)n_snap, G, n_snap, true, s);
  else dgemm_tc(S, 1, n_dof, S, 1, n_dof, w, n_dof, (int)n_snap, (int)n_snap, G, n_snap, true, s);
  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hc
