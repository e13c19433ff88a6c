// Solver workspace and entry points (hc_solver.cu).
#pragma once

#include "hc_internal.cuh"

namespace hc {

struct Work {
  explicit Work(long long nvox);
  DBuf<double2> x, xt, r, rt, d, b;                    // Newton state / residual / step
  DBuf<double2> kr, khat, kp, kv, ks, kt, kph, ksh;    // BiCGStab vectors
  DBuf<double> cprev;                                  // c_prev per voxel
  DBuf<double> part;                                   // reduction partials
  std::vector<double> parth;
  DBuf<double2> xprev_store;
  DBuf<double> npl_tmp;
};

Work& work(Operator& op);
double dot(Operator& op, const double2* a, const double2* b, cudaStream_t s);
double norm_checked(Operator& op, const double2* a, int mask, cudaStream_t s);
int bicgstab_dev(Operator& op, const double2* b, double2* x, double inv_dt, int mode, double rtol,
                 int maxit, cudaStream_t s);
int bicgstab(Operator& op, const double2* b, double2* x, double inv_dt, int mode, double rtol,
             int maxit, cudaStream_t s);
void newton_grid(Operator& op, const double* npl, double dt, double mu, const hc_solver_config& cfg,
                 hc_newton_stats& st, cudaStream_t s);
void initial_potential_grid(Operator& op, const double* npl, double mu, const hc_solver_config& cfg,
                            hc_newton_stats& st, cudaStream_t s);
void step_grid(Operator& op, double* npl, double dt_suggest, double mu, const hc_solver_config& cfg,
               hc_newton_stats& st, cudaStream_t s);

}  // namespace hc
