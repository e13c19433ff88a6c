// Solver workspace and entry points (hc_solver.cu).
#pragma once

#include <vector>

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

// Builds a CUDA graph from captured stream segments and conditional (WHILE / IF) nodes:
// capture() appends whatever the callback launches after the current leaf nodes,
// cond() appends a conditional node and returns its body graph (build it with a child
// builder).  Used for the device-resident Newton solve (hc_solver.cu).
struct GraphBuilder {
  cudaStream_t s;
  cudaGraph_t g;
  std::vector<cudaGraphNode_t> deps;
  template <class F>
  void capture(F&& f) {
    HC_CUDA(cudaStreamBeginCaptureToGraph(s, g, deps.empty() ? nullptr : deps.data(), nullptr, deps.size(),
                                          cudaStreamCaptureModeThreadLocal));
    f();
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* d = nullptr;
    size_t nd = 0;
    HC_CUDA(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &d, &nd));
    std::vector<cudaGraphNode_t> leaf(d, d + nd);
    cudaGraph_t out;
    HC_CUDA(cudaStreamEndCapture(s, &out));
    deps.swap(leaf);
  }
  cudaGraphConditionalHandle handle(unsigned def) {
    cudaGraphConditionalHandle h;
    HC_CUDA(cudaGraphConditionalHandleCreate(&h, g, def, cudaGraphCondAssignDefault));
    return h;
  }
  cudaGraph_t cond(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    HC_CUDA(cudaGraphAddNode(&node, g, deps.empty() ? nullptr : deps.data(), deps.size(), &np));
    deps.assign(1, node);
    return np.conditional.phGraph_out[0];
  }
};

// Appends a whole BiCGStab solve (init, WHILE node over iterations, status check) to
// the graph under construction: rtol is read from *rtol_dev; on breakdown / budget
// exhaustion ns[NS_STATUS] becomes 2, the iterations are added to ns[NS_KITERS].
enum { NS_NORM0, NS_TOL, NS_NORM, NS_IT, NS_STATUS, NS_ALPHA, NS_NTRY, NS_ACC, NS_H, NS_KITERS,
       NS_LINTOL, NS_REBUILD, NS_WHY, NS_N };
void krylov_append(Operator& op, GraphBuilder& gb, const double2* b, double2* x, double inv_dt, int mode,
                   const double* rtol_dev, int maxit, double* ns);
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
