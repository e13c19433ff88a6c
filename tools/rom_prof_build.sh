#!/bin/bash
# Scratch: build paper_1704_04139_b200/csrc/prof/libhalfcell_prof.so, the library with
# per-phase globaltimer accumulators in k_rom_run (run with HC_LIB=<that .so>; prints ROMPROF)
set -e
cd "$(dirname "$0")/../paper_1704_04139_b200/csrc"
mkdir -p prof
python3 - <<'PY'
s = open('hc_rom.cu').read()
parts = s.split('cl.sync();')
out = parts[0]
for i, p in enumerate(parts[1:]):
    out += 'cl.sync(); HC_PROF(%d);' % min(i, 5) + p
s = out
gi = s.rfind('__global__', 0, s.index('k_rom_run('))
s = s[:gi] + '''__device__ unsigned long long g_rom_prof[8];
__device__ __forceinline__ unsigned long long gtimer() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
#define HC_PROF(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { const unsigned long long t_ = gtimer(); g_rom_prof[i] += t_ - t_prev; t_prev = t_; } } while (0)
''' + s[gi:]
s = s.replace('  const int tid = threadIdx.x, nt = blockDim.x;', '  const int tid = threadIdx.x, nt = blockDim.x;\n  unsigned long long t_prev = gtimer();', 1)
s = s.replace('        if (tid < 32) {   // pivots, forward, backward on one warp', '''        unsigned long long tl_ = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) { tl_ = gtimer(); g_rom_prof[6] += tl_ - t_prev; }
        if (tid < 32) {   // pivots, forward, backward on one warp''', 1)
s = s.replace('''            flag[1] = dc == dc && dp == dp;
          }
        }''', '''            flag[1] = dc == dc && dp == dp;
          }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) g_rom_prof[7] += gtimer() - tl_;''', 1)
s = s.replace('''  HC_CUDA(cudaStreamSynchronize(s));
}

}  // namespace hc''', '''  HC_CUDA(cudaStreamSynchronize(s));
  unsigned long long h[8];
  cudaMemcpyFromSymbol(h, g_rom_prof, sizeof h);
  fprintf(stderr, "ROMPROF n_steps=%d phases %.1f %.1f %.1f %.1f %.1f %.1f | E: LU+copy %.1f trisolve %.1f (ms)\\n", (int)n_steps,
          h[0] / 1e6, h[1] / 1e6, h[2] / 1e6, h[3] / 1e6, h[4] / 1e6, h[5] / 1e6, h[6] / 1e6, h[7] / 1e6);
  unsigned long long z[8] = {};
  cudaMemcpyToSymbol(g_rom_prof, z, sizeof z);
}

}  // namespace hc''')
open('prof/hc_rom_prof.cu', 'w').write('#include <cstdio>\n' + s)
PY
nvcc -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -I. -c prof/hc_rom_prof.cu -o prof/hc_rom_prof.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o prof/libhalfcell_prof.so hc_operator.o hc_amg.o hc_solver.o hc_krylov.o hc_capi.o hc_pod.o prof/hc_rom_prof.o -lcudart
