// Aggregation multigrid data structures (see hc_amg.cu).
#pragma once

#include "hc_internal.cuh"

namespace hc {

struct AmgLevel {
  int n = 0;
  long long nnz = 0;
  DBuf<int32_t> rowptr, col;
  DBuf<double> val, dinv;
  DBuf<int32_t> ch_ptr, ch;   // children (previous level unknowns, or fine voxels for level 1)
  DBuf<int32_t> parent;       // unknown -> next coarser unknown
  DBuf<double> x, x2, b, res;
  std::vector<int32_t> h_rowptr, h_col;  // setup only
};

struct AmgBlock {
  int field = 0;                  // 0: c block of T J, 1: phi block of J
  std::vector<AmgLevel> levels;   // levels[0] is aggregation level 1
  DBuf<int32_t> agg1;             // fine voxel -> level-1 unknown, -1 outside the field
  DBuf<double> fine_dinv;         // fine inverse diagonal
  DBuf<double> dense;             // coarsest LU
  DBuf<int> piv;
};

struct Amg {
  AmgBlock blk[2];
  int coarse_max = 256;
  int nu = 2;
  double omega = 0.6;
  DBuf<double2> t, e, zp, rr;
};

Amg* build_amg(const Operator& op);
void amg_update(Operator& op, double inv_dt, int blocks, cudaStream_t s);  // blocks: 1 c, 2 phi
void amg_apply(Operator& op, const double2* r, double2* z, double inv_dt, int mode, cudaStream_t s);

}  // namespace hc
