// POD snapshot Gram matrix G = S^T diag(w) S (method of snapshots, SPEC mor.pod),
// the only dense contraction of the path.  S is n_dof x n_snap column-major fp64.
//
// FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): each CTA owns a 64x64 tile of
// G and a slice of the DOF dimension (split-K); slices are reduced in a fixed
// order afterwards so the result is deterministic.
#include <algorithm>

#include "hc_internal.cuh"

namespace hc {

namespace {
constexpr int BT = 64;   // tile of G
constexpr int KC = 32;   // DOF chunk staged in shared memory
constexpr int NW = 8;    // warps per CTA: 4 (rows of 16) x 2 (cols of 32)

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// part[z][i][j] = sum_{k in slice z} S[k][i] w[k] S[k][j]   (i, j in the CTA tile)
__global__ void __launch_bounds__(NW * 32) k_gram(const double* __restrict__ S,
                                                  const double* __restrict__ w, long long n_dof,
                                                  int n, long long k_per, double* __restrict__ part) {
  __shared__ double As[BT][KC + 1];
  __shared__ double Bs[BT][KC + 1];
  const int ti = blockIdx.x, tj = blockIdx.y, z = blockIdx.z;
  const int i0 = ti * BT, j0 = tj * BT;
  const long long k_begin = (long long)z * k_per;
  const long long k_end = min(n_dof, k_begin + k_per);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wr = warp >> 1, wc = warp & 1;     // warp tile: rows wr*16 .. +16, cols wc*32 .. +32
  const int g = lane >> 2, tq = lane & 3;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (long long k0 = k_begin; k0 < k_end; k0 += KC) {
    // stage: As[i][kk] = S[k0+kk][i0+i] * w, Bs[j][kk] = S[k0+kk][j0+j]
    for (int e = threadIdx.x; e < BT * KC; e += blockDim.x) {
      int col = e / KC, kk = e % KC;
      long long k = k0 + kk;
      double wk = (k < k_end) ? (w ? w[k] : 1.0) : 0.0;
      int gi = i0 + col, gj = j0 + col;
      As[col][kk] = (k < k_end && gi < n) ? S[(long long)gi * n_dof + k] * wk : 0.0;
      Bs[col][kk] = (k < k_end && gj < n) ? S[(long long)gj * n_dof + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < KC; ks += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) af[a] = As[wr * 16 + a * 8 + g][ks + tq];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = Bs[wc * 32 + b * 8 + g][ks + tq];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
  double* out = part + (long long)z * n * n;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int i = i0 + wr * 16 + a * 8 + g;
      int j = j0 + wc * 32 + b * 8 + tq * 2;
      if (i < n && j < n) out[(long long)j * n + i] = acc[a][b][0];
      if (i < n && j + 1 < n) out[(long long)(j + 1) * n + i] = acc[a][b][1];
    }
}

__global__ void k_reduce_parts(long long nn, int nz, const double* __restrict__ part,
                               double* __restrict__ G) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= nn) return;
  double s = 0.0;
  for (int z = 0; z < nz; ++z) s += part[(long long)z * nn + e];
  G[e] = s;
}
}  // namespace

void pod_gram(const double* S, const double* w, long long n_dof, long long n_snap, double* G,
              cudaStream_t s) {
  if (n_snap == 0) return;
  int n = (int)n_snap;
  int tiles = (n + BT - 1) / BT;
  int sms = 148;
  int dev = 0;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  long long want = std::max<long long>(1, (2LL * sms + tiles * tiles - 1) / (tiles * tiles));
  long long k_per = (n_dof + want - 1) / want;
  k_per = ((k_per + KC - 1) / KC) * KC;
  if (k_per == 0) k_per = KC;
  int nz = (int)std::max<long long>(1, (n_dof + k_per - 1) / k_per);
  DBuf<double> part((size_t)nz * n * n);
  dim3 grid(tiles, tiles, nz);
  k_gram<<<grid, NW * 32, 0, s>>>(S, w, n_dof, n, k_per, part.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  long long nn = (long long)n * n;
  k_reduce_parts<<<(int)((nn + 255) / 256), 256, 0, s>>>(nn, nz, part.p, G); HC_COUNT();
  HC_CHECK_LAUNCH();
  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hc
