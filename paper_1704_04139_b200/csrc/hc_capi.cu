// extern "C" entry points of libhalfcell_b200 (include/halfcell_b200.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <tuple>
#include <vector>

#include "hc_amg.cuh"
#include "hc_solver.cuh"

namespace hc {
std::atomic<unsigned long long> g_launch_count{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HC_PDL");
    return !e || atoi(e) != 0;
  }();
  return on;
}
thread_local unsigned long long t_launch_count = 0;
Operator* create_operator(const uint8_t* labels_host, int nx, int ny, int nz, double voxel_um,
                          const hc_params& hp);
void pod_gram(const double* S, const double* w, long long n_dof, long long n_snap, double* G,
              cudaStream_t s, bool rows);
void dgemm_tc(const double* A, long long sa_k, long long sa_i, const double* B, long long sb_k, long long sb_j,
              const double* w, long long K, int M, int N, double* C, long long ldc, bool sym, cudaStream_t s);
double dmma_peak_tflops(cudaStream_t s);
void restricted_eval(const Operator& op, int n_rows, int n_s, const int32_t* f_kind, const int32_t* f_dof,
                     const int32_t* f_slot, const int32_t* row_ptr, const int32_t* row_face,
                     const double* row_coef, const double* xs, const double* npl, double beta, double* out,
                     double* jac, cudaStream_t s);
void rom_run(const Operator& op, const hc_rom* rom, int n_par, double* xt, double* npl, const double* mus_dev,
             double dt, int32_t n_steps, double rtol, int32_t max_iter, int32_t refresh, int32_t jac_steps,
             double* qoi, int32_t* iters, double* xt_steps, int32_t* status_host, cudaStream_t s);

Operator::~Operator() {
  destroy_krylov_graphs(kg);
  destroy_newton_graph(ng);
  delete tma;
  delete amg;
  delete work;
  if (stream) cudaStreamDestroy(stream);
  if (ev_in) cudaEventDestroy(ev_in);
  if (ev_out) cudaEventDestroy(ev_out);
}

// Runs solver work on the operator's private stream, ordered after the
// caller's stream and before anything the caller enqueues afterwards.
struct StreamJoin {
  Operator& op;
  cudaStream_t caller;
  StreamJoin(Operator& o, cudaStream_t c) : op(o), caller(c) {
    HC_CUDA(cudaEventRecord(op.ev_in, caller));
    HC_CUDA(cudaStreamWaitEvent(op.stream, op.ev_in, 0));
  }
  ~StreamJoin() {
    cudaEventRecord(op.ev_out, op.stream);
    cudaStreamWaitEvent(caller, op.ev_out, 0);
  }
};
}  // namespace hc

using namespace hc;

static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return HC_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HC_ERR_CUDA;
  }
}

static cudaStream_t S(void* s) { return (cudaStream_t)s; }

namespace {
// L2 flush by READING a buffer larger than L2: leaves L2 full of clean lines, so the
// timed kernel does not pay for write-backs of a dirty flush buffer
__global__ void k_flush_read(long long n, const double4* __restrict__ buf, double* __restrict__ sink) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double4 q = buf[i];
    s += q.x + q.y + q.z + q.w;
  }
  if (s == 12345.678) sink[0] = s;  // practically never; keeps the loads alive
}

// streaming calibration: read one double2 and write one double2 per voxel (the
// minimum traffic of J v), timed like the stencils to give the practical roofline
__global__ void k_stream_copy(long long n, const double2* __restrict__ a, double2* __restrict__ b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void k_first_nonfinite(long long n, const double* __restrict__ a,
                                  unsigned long long* __restrict__ first) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && !isfinite(a[i])) atomicMin(first, (unsigned long long)i);
}
}  // namespace

extern "C" {

const char* hc_last_error(void) { return g_err.c_str(); }

int hc_device_count(int* out) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *out = n;
  });
}

int hc_operator_create(const uint8_t* labels_host, int32_t nx, int32_t ny, int32_t nz,
                       double voxel_size_um, const hc_params* params, hc_operator** out) {
  return guarded([&] {
    if (!labels_host || !params || !out) throw Error(HC_ERR_ARGUMENT, "null argument");
    *out = (hc_operator*)create_operator(labels_host, nx, ny, nz, voxel_size_um, *params);
  });
}

int hc_operator_destroy(hc_operator* op) {
  return guarded([&] { delete (Operator*)op; });
}

int hc_operator_set_params(hc_operator* opq, const hc_params* params) {
  return guarded([&] {
    if (!opq || !params) throw Error(HC_ERR_ARGUMENT, "null argument");
    Operator& op = *(Operator*)opq;
    set_params(op, *params);
    // everything derived from the old parameters: captured graphs hold DevParams by value,
    // the multigrid hierarchy its Galerkin values
    destroy_krylov_graphs(op.kg);
    op.kg = nullptr;
    destroy_newton_graph(op.ng);
    op.ng = nullptr;
    delete op.amg;
    op.amg = nullptr;
    delete op.work;
    op.work = nullptr;
  });
}

int hc_operator_info(const hc_operator* op, hc_info* out) {
  return guarded([&] { *out = ((const Operator*)op)->info; });
}

int hc_operator_export(const hc_operator* opq, int32_t what, int64_t* out) {
  return guarded([&] {
    const Operator& op = *(const Operator*)opq;
    const long long nvox = op.P.nvox, nc = op.info.n_c;
    auto get = [](const DBuf<int32_t>& b, long long n) {
      std::vector<int32_t> h(n);
      if (n) HC_CUDA(cudaMemcpy(h.data(), b.p, n * 4, cudaMemcpyDeviceToHost));
      return h;
    };
    if (what == 0 || what == 1) {
      auto h = get(what == 0 ? op.cdof : op.pdof, nvox);
      for (long long i = 0; i < nvox; ++i) out[i] = h[i];
      return;
    }
    if (what == 2) {
      auto h = get(op.plated_vox, op.info.n_plated);
      for (size_t i = 0; i < h.size(); ++i) out[i] = h[i];
      return;
    }
    auto cd = get(op.cdof, nvox), pd = get(op.pdof, nvox);
    if (what == 3) {
      long long k = 0;
      for (long long i = 0; i < nvox; ++i)
        if (pd[i] < 0) out[k++] = i;
      return;
    }
    if (what >= 4 && what <= 6) {
      long long off = what == 4 ? 0 : (what == 5 ? op.info.n_bv : op.info.n_bv + op.info.n_ce);
      long long n = what == 4 ? op.info.n_bv : (what == 5 ? op.info.n_ce : op.info.n_strip);
      std::vector<int32_t> so(n), el(n), slot(n);
      if (n) {
        HC_CUDA(cudaMemcpy(so.data(), op.if_solid.p + off, n * 4, cudaMemcpyDeviceToHost));
        HC_CUDA(cudaMemcpy(el.data(), op.if_el.p + off, n * 4, cudaMemcpyDeviceToHost));
        HC_CUDA(cudaMemcpy(slot.data(), op.if_slot.p + off, n * 4, cudaMemcpyDeviceToHost));
      }
      for (long long i = 0; i < n; ++i) {
        if (what == 4) {  // xc_gr, xc_el, xp_gr, xp_el
          out[i] = cd[so[i]];
          out[n + i] = cd[el[i]];
          out[2 * n + i] = nc + pd[so[i]];
          out[3 * n + i] = nc + pd[el[i]];
        } else if (what == 5) {  // xp_fo, xc_el, xp_el
          out[i] = nc + pd[so[i]];
          out[n + i] = cd[el[i]];
          out[2 * n + i] = nc + pd[el[i]];
        } else {  // xp_pl, xc_el, xp_el, slot
          out[i] = nc + pd[so[i]];
          out[n + i] = cd[el[i]];
          out[2 * n + i] = nc + pd[el[i]];
          out[3 * n + i] = slot[i];
        }
      }
      return;
    }
    if (what == 7) {
      long long n = op.info.n_elel;
      auto lo = get(op.elel_lo, n), hi = get(op.elel_hi, n);
      for (long long i = 0; i < n; ++i) {
        out[i] = cd[lo[i]];
        out[n + i] = cd[hi[i]];
        out[2 * n + i] = nc + pd[lo[i]];
        out[3 * n + i] = nc + pd[hi[i]];
      }
      return;
    }
    throw Error(HC_ERR_ARGUMENT, "unknown export selector");
  });
}

int hc_apply(hc_operator* opq, int32_t part, const double* x, const double* n_pl, double mu,
             double beta, double* out, void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    cudaStream_t s = S(stream);
    const long long ntot = op.info.n_c + op.info.n_p;
    int parts = 0;
    switch (part) {
      case 0: parts = PART_LIN | PART_BV | PART_1C | PART_BND; break;
      case 1: parts = PART_BV; break;
      case 2: parts = PART_1C; break;
      case 3: parts = PART_LIN; break;
      case 4: parts = 0; break;
      case 5: parts = PART_BND; mu = 1.0; break;
      default: throw Error(HC_ERR_ARGUMENT, "unknown operator part");
    }
    scatter_packed(op, x, op.xg.p, true, s);
    residual_grid(op, op.xg.p, n_pl, mu, beta, parts, nullptr, 0.0, op.outg.p, s);
    gather_packed(op, op.outg.p, out, s);
    if (part == 0 && ntot) {
      DBuf<unsigned long long> first(1);
      HC_CUDA(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), s));
      k_first_nonfinite<<<(int)((ntot + 255) / 256), 256, 0, s>>>(ntot, out, first.p); HC_COUNT();
      HC_CHECK_LAUNCH();
      unsigned long long f = 0;
      HC_CUDA(cudaMemcpyAsync(&f, first.p, sizeof(f), cudaMemcpyDeviceToHost, s));
      HC_CUDA(cudaStreamSynchronize(s));
      if (f != ~0ULL) {
        int32_t vox = 0;
        const DBuf<int32_t>& m = (long long)f < op.info.n_c ? op.c_vox : op.p_vox;
        long long k = (long long)f < op.info.n_c ? (long long)f : (long long)f - op.info.n_c;
        HC_CUDA(cudaMemcpy(&vox, m.p + k, 4, cudaMemcpyDeviceToHost));
        long long z = vox / op.P.nxy, rem = vox % op.P.nxy, y = rem / op.P.nx, xx = rem % op.P.nx;
        char msg[128];
        snprintf(msg, sizeof msg, "operator produced a non-finite value at voxel (%lld, %lld, %lld)",
                 xx, y, z);
        throw Error(HC_ERR_NUMERICS, msg);
      }
    }
  });
}

int hc_jvp(hc_operator* opq, const double* x, const double* n_pl, double beta, double inv_dt,
           const double* v, double* out, void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    cudaStream_t s = S(stream);
    scatter_packed(op, x, op.xg.p, true, s);
    linearize(op, op.xg.p, n_pl, beta, s);
    scatter_packed(op, v, op.vg.p, false, s);
    jvp_grid(op, op.vg.p, inv_dt, 1 | 4, op.outg.p, s);
    gather_packed(op, op.outg.p, out, s);
  });
}

}  // extern "C"

// Host assembly of A_lin (operator.py:121-221, coo -> csr: duplicates summed) or of the
// analytic Jacobian A_lin + J_nl (operator.py:458-471: scipy csr + csr, exact zeros of the
// sum dropped).
static void assemble_csr(Operator& op, const double* x, const double* n_pl, double beta, bool with_nl,
                         int64_t* nnz_out, int64_t* row_ptr, int64_t* col_idx, double* values) {
  {
    const DevParams& P = op.P;
    const long long nvox = P.nvox, nc = op.info.n_c, n = op.info.n_c + op.info.n_p;
    if (with_nl) {
      scatter_packed(op, x, op.xg.p, true, 0);
      linearize(op, op.xg.p, n_pl, beta, 0);
    }
    HC_CUDA(cudaDeviceSynchronize());
    std::vector<uint8_t> lab(nvox);
    std::vector<int32_t> cd(nvox), pd(nvox), so(op.n_if), el(op.n_if);
    std::vector<int8_t> kd(op.n_if);
    std::vector<double> coef(3 * op.n_if), w(nvox);
    HC_CUDA(cudaMemcpy(lab.data(), op.labels.p, nvox, cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(cd.data(), op.cdof.p, nvox * 4, cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(pd.data(), op.pdof.p, nvox * 4, cudaMemcpyDeviceToHost));
    if (with_nl) HC_CUDA(cudaMemcpy(w.data(), op.inv_c.p, nvox * 8, cudaMemcpyDeviceToHost));
    if (op.n_if && with_nl) {
      HC_CUDA(cudaMemcpy(so.data(), op.if_solid.p, op.n_if * 4, cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(el.data(), op.if_el.p, op.n_if * 4, cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(kd.data(), op.if_kind.p, op.n_if, cudaMemcpyDeviceToHost));
      HC_CUDA(cudaMemcpy(coef.data(), op.if_coef.p, 3 * op.n_if * 8, cudaMemcpyDeviceToHost));
    }
    std::vector<std::map<int64_t, double>> rows(n);
    auto add = [&](long long r, long long c, double v) { rows[r][c] += v; };
    auto xc = [&](long long v) { return (long long)cd[v]; };
    auto xp = [&](long long v) { return nc + pd[v]; };
    const double gF2 = P.gF2, gM = P.t_plus * P.kappa * gF2;
    auto gnd = [&](long long v) { return pd[v] < 0; };
    long long nx = P.nx, ny = P.ny, nz = P.nz;
    for (int axis = 0; axis < 3; ++axis) {
      for (long long z = 0; z < nz; ++z)
        for (long long y = 0; y < ny; ++y)
          for (long long xx = 0; xx < nx; ++xx) {
            if ((axis == 0 && z + 1 >= nz) || (axis == 1 && y + 1 >= ny) || (axis == 2 && xx + 1 >= nx))
              continue;
            long long lo = (z * ny + y) * nx + xx;
            long long hi = lo + (axis == 0 ? nx * ny : (axis == 1 ? nx : 1));
            uint8_t a = lab[lo], b = lab[hi];
            uint8_t k = kind_of(a, b);
            bool gl = gnd(lo), gh = gnd(hi);
            if (gl && gh) continue;
            if (gl || gh) {
              if (k == K_CONT || k == K_CONTACT) {
                long long live = gl ? hi : lo;
                add(xp(live), xp(live), 2.0 * P.sig[a] * P.sig[b] / (P.sig[a] + P.sig[b]) * gF2);
              }
              continue;
            }
            auto sym = [&](long long i, long long j, double g) {
              add(i, i, g); add(i, j, -g); add(j, j, g); add(j, i, -g);
            };
            if (k == K_CONT) {
              if (a == GR) {
                sym(xc(lo), xc(hi), P.d_gr * P.inv_h2);
                sym(xp(lo), xp(hi), P.sigma_gr * gF2);
              } else if (a == EL) {
                sym(xc(lo), xc(hi), P.d_el * P.inv_h2);
                sym(xp(lo), xp(hi), P.kappa * gF2);
                add(xc(lo), xp(lo), gM); add(xc(lo), xp(hi), -gM);
                add(xc(hi), xp(hi), gM); add(xc(hi), xp(lo), -gM);
              } else {
                sym(xp(lo), xp(hi), P.sig[a] * gF2);
              }
            } else if (k == K_CONTACT) {
              sym(xp(lo), xp(hi), 2.0 * P.sig[a] * P.sig[b] / (P.sig[a] + P.sig[b]) * gF2);
            }
          }
    }
    // A_lin done: snapshot as its own summed matrix, then add the nonlinear part
    std::vector<std::map<int64_t, double>> nl(with_nl ? n : 0);
    auto addn = [&](long long r, long long c, double v) { nl[r][c] += v; };
    for (long long f = 0; with_nl && f < op.n_if; ++f) {
      long long s_ = so[f], e = el[f];
      double ca = coef[f], cb = coef[op.n_if + f], cg = coef[2 * op.n_if + f];
      if (kd[f] == IF_BV) {
        const long long rs[4] = {xc(s_), xp(s_), xc(e), xp(e)};
        const double sg[4] = {1, 1, -1, -1};
        for (int q = 0; q < 4; ++q) {
          addn(rs[q], xc(s_), sg[q] * ca);
          addn(rs[q], xc(e), sg[q] * cb);
          addn(rs[q], xp(s_), sg[q] * cg);
          addn(rs[q], xp(e), -sg[q] * cg);
        }
      } else if (kd[f] == IF_CE) {
        const long long rs[3] = {xp(s_), xc(e), xp(e)};
        const double sg[3] = {1, -1, -1};
        for (int q = 0; q < 3; ++q) {
          addn(rs[q], xp(s_), sg[q] * cg);
          addn(rs[q], xp(e), -sg[q] * cg);
        }
      } else {
        const long long rs[3] = {xp(s_), xc(e), xp(e)};
        const double sg[3] = {1, -1, -1};
        for (int q = 0; q < 3; ++q) {
          addn(rs[q], xc(e), sg[q] * cb);
          addn(rs[q], xp(s_), sg[q] * cg);
          addn(rs[q], xp(e), -sg[q] * cg);
        }
      }
    }
    if (with_nl) {
      std::vector<int32_t> lo(op.info.n_elel), hi(op.info.n_elel);
      if (op.info.n_elel) {
        HC_CUDA(cudaMemcpy(lo.data(), op.elel_lo.p, lo.size() * 4, cudaMemcpyDeviceToHost));
        HC_CUDA(cudaMemcpy(hi.data(), op.elel_hi.p, hi.size() * 4, cudaMemcpyDeviceToHost));
      }
      for (size_t f = 0; f < lo.size(); ++f) {
        long long i = lo[f], j = hi[f];
        double dqi = -w[i], dqj = w[j];   // -gX/c_i, gX/c_j
        const long long rs[4] = {xp(i), xp(j), xc(i), xc(j)};
        const double sg[4] = {-1.0, 1.0, -P.t_plus, P.t_plus};
        for (int q = 0; q < 4; ++q) {
          addn(rs[q], xc(i), sg[q] * dqi);
          addn(rs[q], xc(j), sg[q] * dqj);
        }
      }
    }
    long long nnz = 0;
    for (long long r = 0; r < n; ++r) {
      if (with_nl) {
        for (auto& kv : nl[r]) rows[r][kv.first] += kv.second;
        for (auto it = rows[r].begin(); it != rows[r].end();) {
          if (it->second == 0.0) it = rows[r].erase(it); else ++it;
        }
      }
      nnz += (long long)rows[r].size();
    }
    *nnz_out = nnz;
    if (!row_ptr) return;
    long long k = 0;
    row_ptr[0] = 0;
    for (long long r = 0; r < n; ++r) {
      for (auto& kv : rows[r]) {
        col_idx[k] = kv.first;
        if (values) values[k] = kv.second;
        ++k;
      }
      row_ptr[r + 1] = k;
    }
  }
}

static void load_prev(Operator& op, const double* x_prev, cudaStream_t s);
// Clears the Newton trace / source settings of an operator on scope exit.
struct TraceScope {
  Operator& op;
  ~TraceScope() {
    op.iter_out = nullptr;
    op.iter_max = 0;
    op.trace_norms = false;
    op.src = nullptr;
  }
};

extern "C" {

int hc_jacobian_csr(hc_operator* opq, const double* x, const double* n_pl, double beta,
                    int64_t* nnz_out, int64_t* row_ptr, int64_t* col_idx, double* values) {
  return guarded([&] {
    assemble_csr(*(Operator*)opq, x, n_pl, beta, true, nnz_out, row_ptr, col_idx, values);
  });
}

int hc_lin_csr(hc_operator* opq, int64_t* nnz_out, int64_t* row_ptr, int64_t* col_idx, double* values) {
  return guarded([&] {
    assemble_csr(*(Operator*)opq, nullptr, nullptr, 0.0, false, nnz_out, row_ptr, col_idx, values);
  });
}

int hc_precond_refresh(hc_operator* opq) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    if (op.amg) op.amg->force = true;
  });
}

int hc_strip_face_currents(hc_operator* opq, const double* x, const double* n_pl, double beta,
                           double* out, void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    cudaStream_t s = S(stream);
    if (!op.info.n_strip) return;
    scatter_packed(op, x, op.xg.p, true, s);
    strip_currents(op, op.xg.p, n_pl, beta, out, s);
  });
}

int hc_newton_solve(hc_operator* opq, const double* x_guess, double dt, const double* x_prev,
                    const double* n_pl, double mu, const hc_solver_config* cfg, double* x_out,
                    hc_newton_stats* stats, void* stream) {
  return hc_newton_solve_ex(opq, x_guess, dt, x_prev, n_pl, mu, cfg, nullptr, nullptr, 0, nullptr, 0,
                            x_out, stats, stream);
}

int hc_newton_solve_ex(hc_operator* opq, const double* x_guess, double dt, const double* x_prev,
                       const double* n_pl, double mu, const hc_solver_config* cfg, const double* source,
                       double* iterates, int32_t max_iterates, double* norms, int32_t max_norms,
                       double* x_out, hc_newton_stats* stats, void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    StreamJoin join(op, S(stream));
    cudaStream_t s = op.stream;
    Work& W = work(op);
    TraceScope trace{op};
    hc_newton_stats st{};
    load_prev(op, x_prev, s);
    if (source) {
      scatter_packed(op, source, op.vg.p, false, s);
      op.src = op.vg.p;
    }
    op.iter_out = iterates;
    op.iter_max = iterates ? std::max(0, max_iterates) : 0;
    op.trace_norms = norms != nullptr;
    for (int attempt = 0;; ++attempt) {
      scatter_packed(op, x_guess, W.x.p, true, s);
      op.krylov_fail_stale = false;
      try {
        newton_grid(op, n_pl, dt, mu, *cfg, st, s);
      } catch (const Error& e) {
        // a Krylov failure on a lagged multigrid hierarchy is the solver's, not the
        // problem's: rebuild the hierarchy and solve again once
        if (e.code != HC_ERR_NONCONVERGENCE || !op.krylov_fail_stale || attempt) throw;
        op.amg->force = true;
        continue;
      }
      break;
    }
    gather_packed(op, W.x.p, x_out, s);
    HC_CUDA(cudaStreamSynchronize(s));
    if (norms)
      for (int i = 0; i < max_norms && i < (int)op.norm_log.size(); ++i) norms[i] = op.norm_log[i];
    if (stats) *stats = st;
  });
}

int hc_solve_initial_potential(hc_operator* opq, const double* x0, const double* n_pl, double mu,
                               const hc_solver_config* cfg, double* x_out, hc_newton_stats* stats,
                               void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    StreamJoin join(op, S(stream));
    cudaStream_t s = op.stream;
    Work& W = work(op);
    hc_newton_stats st{};
    scatter_packed(op, x0, W.x.p, true, s);
    initial_potential_grid(op, n_pl, mu, *cfg, st, s);
    gather_packed(op, W.x.p, x_out, s);
    HC_CUDA(cudaStreamSynchronize(s));
    if (stats) *stats = st;
  });
}

int hc_step(hc_operator* opq, double* x, double* n_pl, double t, double dt_suggest, double mu,
            const hc_solver_config* cfg, hc_newton_stats* stats, void* stream) {
  return hc_step_ex(opq, x, n_pl, t, dt_suggest, mu, cfg, nullptr, 0, stats, stream);
}

int hc_step_ex(hc_operator* opq, double* x, double* n_pl, double t, double dt_suggest, double mu,
               const hc_solver_config* cfg, double* iterates, int32_t max_iterates, hc_newton_stats* stats,
               void* stream) {
  (void)t;
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    StreamJoin join(op, S(stream));
    cudaStream_t s = op.stream;
    Work& W = work(op);
    TraceScope trace{op};
    op.iter_out = iterates;
    op.iter_max = iterates ? std::max(0, max_iterates) : 0;
    hc_newton_stats st{};
    scatter_packed(op, x, W.x.p, true, s);
    step_grid(op, n_pl, dt_suggest, mu, *cfg, st, s);
    gather_packed(op, W.x.p, x, s);
    HC_CUDA(cudaStreamSynchronize(s));
    if (stats) *stats = st;
  });
}

int hc_step_host(hc_operator* opq, double* x_host, double* n_pl_host, double t, double dt_suggest,
                 double mu, const hc_solver_config* cfg, hc_newton_stats* stats) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    const long long ntot = op.info.n_c + op.info.n_p, npl = op.info.n_plated;
    if (op.host_x.n < (size_t)ntot) op.host_x.alloc(std::max<long long>(ntot, 1));
    if (op.host_npl.n < (size_t)std::max<long long>(npl, 1)) op.host_npl.alloc(std::max<long long>(npl, 1));
    cudaStream_t s = op.stream;
    HC_CUDA(cudaMemcpyAsync(op.host_x.p, x_host, ntot * 8, cudaMemcpyHostToDevice, s));
    if (npl) HC_CUDA(cudaMemcpyAsync(op.host_npl.p, n_pl_host, npl * 8, cudaMemcpyHostToDevice, s));
    Work& W = work(op);
    hc_newton_stats st{};
    scatter_packed(op, op.host_x.p, W.x.p, true, s);
    step_grid(op, op.host_npl.p, dt_suggest, mu, *cfg, st, s);
    gather_packed(op, W.x.p, op.host_x.p, s);
    HC_CUDA(cudaMemcpyAsync(x_host, op.host_x.p, ntot * 8, cudaMemcpyDeviceToHost, s));
    if (npl) HC_CUDA(cudaMemcpyAsync(n_pl_host, op.host_npl.p, npl * 8, cudaMemcpyDeviceToHost, s));
    HC_CUDA(cudaStreamSynchronize(s));
    if (stats) *stats = st;
    (void)t;
  });
}

int hc_launch_count(int64_t* out) {
  return guarded([&] { *out = (int64_t)g_launch_count.load(); });
}

int hc_time_kernels(hc_operator* opq, const double* x, const double* n_pl, double beta,
                    double inv_dt, int32_t iters, int64_t flush_bytes, double* ms_out,
                    void* stream) {
  return guarded([&] {
    Operator& op = *(Operator*)opq;
    cudaStream_t s = S(stream);
    scatter_packed(op, x, op.xg.p, true, s);
    linearize(op, op.xg.p, n_pl, beta, s);
    Work& W = work(op);
    HC_CUDA(cudaMemcpyAsync(W.cprev.p, op.inv_c.p, op.P.nvox * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));  // any finite c_prev will do
    DBuf<uint8_t> scratch(flush_bytes > 0 ? (size_t)flush_bytes : 0);
    DBuf<double> sink(1);
    if (scratch.n) HC_CUDA(cudaMemsetAsync(scratch.p, 0, scratch.n, s));
    cudaEvent_t e0, e1;
    HC_CUDA(cudaEventCreate(&e0));
    HC_CUDA(cudaEventCreate(&e1));
    const int parts = PART_LIN | PART_BV | PART_1C | PART_BND | PART_TIME;
    for (int k = 0; k < 5; ++k) {
      double acc = 0.0;
      for (int it = 0; it < iters; ++it) {
        if (scratch.n) {
          k_flush_read<<<4 * op.n_sm, 256, 0, s>>>((long long)(scratch.n / sizeof(double4)),
                                                   (const double4*)scratch.p, sink.p);
        }
        HC_CUDA(cudaEventRecord(e0, s));
        if (k < 2)
          residual_grid(op, op.xg.p, n_pl, -1.0, beta, parts, W.cprev.p, inv_dt, op.outg.p, s,
                        k == 0 ? 1 : 2);
        else if (k < 4)
          jvp_grid(op, op.xg.p, inv_dt, 1 | 4, op.outg.p, s, k == 2 ? 1 : 2);
        else
          k_stream_copy<<<4 * op.n_sm, 256, 0, s>>>(op.P.nvox, op.xg.p, op.outg.p);
        HC_CUDA(cudaEventRecord(e1, s));
        HC_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        HC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        acc += ms;
      }
      ms_out[k] = iters ? acc / iters : 0.0;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int hc_step_batch(hc_operator* const* ops, int32_t n, double* const* x, double* const* n_pl,
                  const double* dt_suggest, const double* mu, const hc_solver_config* cfg,
                  hc_newton_stats* stats, int32_t n_threads) {
  return guarded([&] {
    if (n <= 0) return;
    int dev = 0;
    HC_CUDA(cudaGetDevice(&dev));
    int nt = std::max(1, std::min<int>(n_threads > 0 ? n_threads : 16, n));
    // many cells share the GPU through host threads: the device-resident Newton graph
    // (one host wait per step instead of a few per Newton iteration) measured +25 %
    // here (253 -> 317 cell-steps/s), so it is the default for batches (HC_NEWTON_DEV=0 off)
    const char* nd = getenv("HC_NEWTON_DEV");
    const bool dev_newton = !nd || atoi(nd) != 0;
    std::vector<char> saved(n);
    for (int i = 0; i < n; ++i) {
      saved[i] = ((Operator*)ops[i])->newton_dev;
      ((Operator*)ops[i])->newton_dev = dev_newton;
    }
    if (stats)
      for (int i = 0; i < n; ++i) stats[i] = hc_newton_stats{};
    std::atomic<int> next{0};
    std::mutex m;
    int first_code = HC_OK;
    std::string first_msg;
    auto worker = [&] {
      cudaSetDevice(dev);
      for (int i; (i = next.fetch_add(1)) < n;) {
        try {
          Operator& op = *(Operator*)ops[i];
          Work& W = work(op);
          cudaStream_t s = op.stream;
          hc_newton_stats st{};
          scatter_packed(op, x[i], W.x.p, true, s);
          step_grid(op, n_pl[i], dt_suggest[i], mu[i], *cfg, st, s);
          gather_packed(op, W.x.p, x[i], s);
          HC_CUDA(cudaStreamSynchronize(s));
          if (stats) stats[i] = st;
        } catch (const Error& e) {
          // the failed cell keeps its input state (x[i] is only written on success; n_pl is
          // updated after the Newton solve only) and reports its code in status
          if (stats) stats[i].status = e.code;
          std::lock_guard<std::mutex> g(m);
          if (first_code == HC_OK) { first_code = e.code; first_msg = "cell " + std::to_string(i) + ": " + e.what(); }
        } catch (const std::exception& e) {
          if (stats) stats[i].status = HC_ERR_CUDA;
          std::lock_guard<std::mutex> g(m);
          if (first_code == HC_OK) { first_code = HC_ERR_CUDA; first_msg = e.what(); }
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();
    for (int i = 0; i < n; ++i) ((Operator*)ops[i])->newton_dev = saved[i];
    if (first_code != HC_OK) throw Error(first_code, first_msg);
  });
}

int hc_flush_l2(int64_t bytes, void* stream) {
  return guarded([&] {
    static DBuf<uint8_t> buf;
    static DBuf<double> sink(1);
    if (buf.n < (size_t)bytes) {
      buf.alloc((size_t)bytes);
      HC_CUDA(cudaMemset(buf.p, 0, buf.n));
    }
    int dev = 0, sms = 148;
    HC_CUDA(cudaGetDevice(&dev));
    HC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    k_flush_read<<<4 * sms, 256, 0, S(stream)>>>((long long)(bytes / sizeof(double4)),
                                                 (const double4*)buf.p, sink.p);
    HC_CHECK_LAUNCH();
  });
}

int hc_pod_gram(const double* Sm, const double* w, int64_t n_dof, int64_t n_snap, double* G,
                void* stream) {
  return guarded([&] {
    if (n_dof < 0 || n_snap < 0) throw Error(HC_ERR_ARGUMENT, "negative size");
    pod_gram(Sm, w, n_dof, n_snap, G, S(stream), false);
  });
}

int hc_dgemm(const double* A, int64_t sa_k, int64_t sa_i, const double* B, int64_t sb_k, int64_t sb_j,
             const double* w, int64_t K, int32_t M, int32_t N, double* C, int64_t ldc, void* stream) {
  return guarded([&] {
    if (K < 0 || M < 0 || N < 0 || ldc < N) throw Error(HC_ERR_ARGUMENT, "bad contraction shape");
    if ((M && N && K) && (!A || !B || !C)) throw Error(HC_ERR_ARGUMENT, "null operand");
    dgemm_tc(A, sa_k, sa_i, B, sb_k, sb_j, w, K, M, N, C, ldc, false, S(stream));
  });
}

int hc_dmma_peak(double* tflops, void* stream) {
  return guarded([&] { *tflops = dmma_peak_tflops(S(stream)); });
}

int hc_pod_gram_rows(const double* Sm, const double* w, int64_t n_dof, int64_t n_snap, double* G,
                     void* stream) {
  return guarded([&] {
    if (n_dof < 0 || n_snap < 0) throw Error(HC_ERR_ARGUMENT, "negative size");
    pod_gram(Sm, w, n_dof, n_snap, G, S(stream), true);
  });
}

int hc_restricted_eval(hc_operator* opq, int32_t n_rows, int32_t n_f, int32_t n_s, const int32_t* f_kind,
                       const int32_t* f_dof, const int32_t* f_slot, const int32_t* row_ptr,
                       const int32_t* row_face, const double* row_coef, const double* x_st,
                       const double* n_pl, double beta, double* out, double* jac, void* stream) {
  return guarded([&] {
    if (!opq || n_rows < 0 || n_f < 0 || n_s < 0) throw Error(HC_ERR_ARGUMENT, "bad restricted operator");
    (void)n_f;
    restricted_eval(*(Operator*)opq, n_rows, n_s, f_kind, f_dof, f_slot, row_ptr, row_face, row_coef, x_st,
                    n_pl, beta, out, jac, S(stream));
  });
}

int hc_rom_run(hc_operator* opq, const hc_rom* rom, double* xt, double* n_pl, double mu, double dt,
               int32_t n_steps, double rtol, int32_t max_iter, int32_t refresh, int32_t jac_steps,
               double* qoi, int32_t* iters, double* xt_steps, int32_t* failed_step, void* stream) {
  return guarded([&] {
    if (!opq || !rom || !xt) throw Error(HC_ERR_ARGUMENT, "null argument");
    if (!(dt > 0.0) || n_steps < 0 || max_iter < 1) throw Error(HC_ERR_ARGUMENT, "bad step settings");
    int32_t st[4] = {0, 0, 0, 0};
    DBuf<double> mu_d(1);
    HC_CUDA(cudaMemcpyAsync(mu_d.p, &mu, sizeof(double), cudaMemcpyHostToDevice, S(stream)));
    rom_run(*(Operator*)opq, rom, 1, xt, n_pl, mu_d.p, dt, n_steps, rtol, max_iter, refresh,
            std::max(1, jac_steps), qoi, iters, xt_steps, st, S(stream));
    if (failed_step) *failed_step = st[0] ? st[1] : -1;
    if (st[0] == 1) throw Error(HC_ERR_NONCONVERGENCE, "reduced Newton did not converge");
    if (st[0] == 2) throw Error(HC_ERR_NUMERICS, "reduced Newton produced a non-finite update");
  });
}

int hc_rom_run_batch(hc_operator* opq, const hc_rom* rom, int32_t n_par, double* xt, double* n_pl,
                     const double* mu, double dt, int32_t n_steps, double rtol, int32_t max_iter,
                     int32_t refresh, int32_t jac_steps, double* qoi, int32_t* iters, int32_t* failed_step,
                     void* stream) {
  return guarded([&] {
    if (!opq || !rom || !xt || !mu || n_par < 1) throw Error(HC_ERR_ARGUMENT, "null argument");
    if (!(dt > 0.0) || n_steps < 0 || max_iter < 1) throw Error(HC_ERR_ARGUMENT, "bad step settings");
    std::vector<int32_t> st(4 * (size_t)n_par, 0);
    rom_run(*(Operator*)opq, rom, n_par, xt, n_pl, mu, dt, n_steps, rtol, max_iter, refresh,
            std::max(1, jac_steps), qoi, iters, nullptr, st.data(), S(stream));
    int bad = 0;
    for (int p = 0; p < n_par; ++p) {
      if (failed_step) failed_step[p] = st[4 * p] ? st[4 * p + 1] : -1;
      bad |= st[4 * p];
    }
    if (bad & 2) throw Error(HC_ERR_NUMERICS, "reduced Newton produced a non-finite update");
    if (bad & 1) throw Error(HC_ERR_NONCONVERGENCE, "reduced Newton did not converge");
  });
}

}  // extern "C"

namespace {
__global__ void k_extract_c2(long long n, const double2* __restrict__ x, double* __restrict__ c) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) c[i] = x[i].x;
}
}  // namespace

static void load_prev(Operator& op, const double* x_prev, cudaStream_t s) {
  Work& W = work(op);
  scatter_packed(op, x_prev, op.xg2.p, true, s);
  long long n = op.P.nvox;
  k_extract_c2<<<(int)((n + 255) / 256), 256, 0, s>>>(n, op.xg2.p, W.cprev.p); HC_COUNT();
  HC_CHECK_LAUNCH();
}
