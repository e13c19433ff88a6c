// Scratch probe: TMA 3-D box loads with the helpers of hc_tma.cuh.
// nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1704_04139_b200/csrc tools/tma_probe.cu -o tools/tma_probe
#include <cstdio>
#include <vector>
#include <cudaTypedefs.h>
#include "hc_tma.cuh"

using namespace hc;

namespace hc {
int g_box0 = T_LW; CUtensorMapL2promotion g_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
bool tma_encode(CUtensorMap* m, const void* ptr, int kind, int nx, int ny, int nz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz}, strides[2];
  cuuint32_t box[3] = {(cuuint32_t)g_box0, T_TH, 1}, es[3] = {1, 1, 1};
  strides[0] = nx * 4;
  strides[1] = strides[0] * ny;
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  g_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode -> %d\n", (int)r);
  return r == CUDA_SUCCESS;
}
}  // namespace hc

__global__ void k_glob(const CUtensorMap* gm, int* out, int x, int y, int bytes) {
  __shared__ __align__(128) int tile[T_LN];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(b, bytes);
    tma_load3((unsigned)__cvta_generic_to_shared(tile), gm, x, y, 0, b);
  }
  mbar_wait(b, 0);
  __syncthreads();
  for (int i = threadIdx.x; i < T_LN; i += blockDim.x) out[i] = tile[i];
}
__global__ void k_plain(const __grid_constant__ CUtensorMap m, int* out, int mode) {
  __shared__ __align__(128) int tile[T_LN];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(b, T_LN * 4);
    if (mode >= 1) tma_load3((unsigned)__cvta_generic_to_shared(tile), &m, -1, -1, 0, b);
  }
  if (mode >= 1) mbar_wait(b, 0);
  __syncthreads();
  for (int i = threadIdx.x; i < T_LN; i += blockDim.x) out[i] = tile[i];
}

struct Two {
  CUtensorMap a, b;
};
__global__ void k_struct(const __grid_constant__ Two m, int* out) {
  __shared__ __align__(128) int tile[T_LN];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    mbar_expect_tx(b, T_LN * 4);
    tma_load3((unsigned)__cvta_generic_to_shared(tile), &m.b, 3, 2, 1, b);
  }
  mbar_wait(b, 0);
  __syncthreads();
  for (int i = threadIdx.x; i < T_LN; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int nx = 64, ny = 16, nz = 4;
  std::vector<int> h(nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (int)i + 1;
  int *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, T_LN * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  tma_encode(&m, d, 0, nx, ny, nz);
  std::vector<int> r(T_LN);
  CUtensorMap* gm;
  cudaMalloc(&gm, sizeof(CUtensorMap));
  struct V { int box0; CUtensorMapL2promotion pr; int x, y; } vs[] = {
      {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 4, -1}, {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, -4, 0},
      {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 0, 15}, {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 60, 0},
      {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 2, 0}, {36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 1, 0}};
  for (auto& v : vs) {
    g_box0 = v.box0; g_promo = v.pr;
    CUtensorMap mm;
    tma_encode(&mm, d, 0, nx, ny, nz);
    cudaMemcpy(gm, &mm, sizeof(mm), cudaMemcpyHostToDevice);
    k_glob<<<1, 128>>>(gm, o, v.x, v.y, v.box0 * T_TH * 4);
    cudaError_t e = cudaDeviceSynchronize();
    printf("global map box0 %d promo %d at (%d,%d): %s\n", v.box0, (int)v.pr, v.x, v.y, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(r.data(), o, T_LN * 4, cudaMemcpyDeviceToHost);
    printf("  tile[0] %d tile[1] %d tile[4] %d tile[36] %d\n", r[0], r[1], r[4], r[36]);
  }
  g_box0 = T_LW; g_promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(o, 0xff, T_LN * 4);
    k_plain<<<1, 128>>>(m, o, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("plain mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(r.data(), o, T_LN * 4, cudaMemcpyDeviceToHost);
    printf("  tile[0..3] %d %d %d %d  tile[T_LW+1] %d (expect %d)\n", r[0], r[1], r[2], r[3],
           r[T_LW + 1], h[0]);
  }
  Two t{m, m};
  k_struct<<<1, 128>>>(t, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("struct: %s\n", cudaGetErrorString(e));
  cudaMemcpy(r.data(), o, T_LN * 4, cudaMemcpyDeviceToHost);
  printf("  tile[0] %d (expect %d)\n", r[0], h[(1 * ny + 2) * nx + 3]);
  return 0;
}
