// Internal definitions shared by the halfcell_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/halfcell_b200.h"

namespace hc {

// ---- phases (reference microgen/phases.py:18-26) --------------------------------
enum : uint8_t { EL = 0, GR = 1, PL = 2, FOIL = 3, CW = 4, CC = 5, N_PHASES = 6 };

// ---- interface kinds (reference echem/interfaces.py:23-61, operator.py:39-52) ---
enum : uint8_t { K_CONT = 0, K_BV = 1, K_CE = 2, K_STRIP = 3, K_BLOCK = 4, K_CONTACT = 5, K_FORBID = 6 };

__host__ __device__ inline uint8_t kind_of(uint8_t a, uint8_t b) {
  if (a == b) return K_CONT;
  uint8_t lo = a < b ? a : b, hi = a < b ? b : a;
  // lo < hi
  if (lo == EL) {
    if (hi == GR) return K_BV;
    if (hi == FOIL) return K_CE;
    if (hi == PL) return K_STRIP;
    return K_BLOCK;  // CW, CC
  }
  if (hi == FOIL && (lo == GR || lo == PL)) return K_FORBID;
  return K_CONTACT;
}

// ---- exceptions carried to the C ABI -------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define HC_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::hc::Error(HC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

#define HC_CHECK_LAUNCH() HC_CUDA(cudaGetLastError())

// process-wide count of kernels launched by this library (bench.py's gpu_launches)
extern std::atomic<unsigned long long> g_launch_count;
extern thread_local unsigned long long t_launch_count;   // this thread's launches (captures)
inline void count_launch() {
  g_launch_count.fetch_add(1, std::memory_order_relaxed);
  ++t_launch_count;
}
inline void count_graph_launch(unsigned long long n) {
  g_launch_count.fetch_add(n, std::memory_order_relaxed);
}
// launches recorded while capturing a graph are not kernel executions: undo them
inline void uncount(unsigned long long n) { g_launch_count.fetch_sub(n, std::memory_order_relaxed); }
#define HC_COUNT() (::hc::count_launch())

// ---- device-side parameter block (passed by value to kernels) -------------------
struct DevParams {
  int nx, ny, nz;
  long long nxy, nvox;
  double h;            // m
  double gF2;          // 1 / (F h^2)
  double sc;           // 1 / (F h)
  double inv_h2;       // 1 / h^2
  double d_gr, d_el, t_plus, kappa, sigma_gr;
  double sig[N_PHASES];
  double gX;           // chemical-potential face coefficient (operator.py:225-226)
  double vt;           // 2RT/F
  double i00_grel, i00_ceel, i00_plel, c_gr_max, n_const;
  double drive;        // -1/(F h): b_bnd entry (operator.py:231-233)
  int n_ocp;
  double ocp_soc[HC_MAX_OCP];
  double ocp_v[HC_MAX_OCP];
  // face-coefficient tables indexed [a * 6 + b] (a: row phase, b: neighbour phase);
  // grounded neighbours hold phi = 0, so their closure is the ordinary face formula
  double gP[36];      // phi-row conduction (same phase: sigma_a, contact: harmonic mean) * gF2
  double gC[36];      // c-row diffusion (graphite / electrolyte same-phase faces)
  double gMig[36];    // c-row migration coupling to phi (electrolyte-electrolyte)
  unsigned char ifc[36];  // 1 for interface-kinetics pairs (BV, counter exchange, stripping)
};

// 3-D launch shape of the per-voxel stencil kernels: a warp spans 32 consecutive
// x, a block 32 x 8 in the xy plane, blockIdx.z = z.  No 64-bit index division.
constexpr int VX = 32, VY = 8;
inline dim3 vox_grid(const DevParams& P) {
  return dim3((unsigned)((P.nx + VX - 1) / VX), (unsigned)((P.ny + VY - 1) / VY), (unsigned)P.nz);
}
inline dim3 vox_block() { return dim3(VX, VY, 1); }
__device__ __forceinline__ bool vox_index(const DevParams& P, int& x, int& y, int& z, int& v) {
  x = blockIdx.x * VX + threadIdx.x;
  y = blockIdx.y * VY + threadIdx.y;
  z = blockIdx.z;
  if (x >= P.nx || y >= P.ny) return false;
  v = (z * P.ny + y) * P.nx + x;
  return true;
}

// np.interp on the OCP table (echem/kinetics.py:25-32), clamped at the ends.  The
// segment is found by binary search (the last knot index j <= n-2 with soc[j] <= s),
// the same segment the linear scan of the reference's np.interp picks.
__device__ __host__ inline double ocp_dev(double c, const DevParams& P) {
  double s = c / P.c_gr_max;
  int n = P.n_ocp;
  if (!(s >= P.ocp_soc[0])) return (s != s) ? s : P.ocp_v[0];
  if (s >= P.ocp_soc[n - 1]) return P.ocp_v[n - 1];
  int lo = 0, hi = n - 2;   // invariant: soc[lo] <= s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.ocp_soc[mid] <= s) lo = mid; else hi = mid - 1;
  }
  const int j = lo;
  double slope = (P.ocp_v[j + 1] - P.ocp_v[j]) / (P.ocp_soc[j + 1] - P.ocp_soc[j]);
  return slope * (s - P.ocp_soc[j]) + P.ocp_v[j];
}

// d OCP / d c (echem/kinetics.py:35-42): segment by searchsorted(side=right)-1,
// clipped; zero outside the table range.
__device__ __host__ inline double ocp_slope_dev(double c, const DevParams& P) {
  double s = c / P.c_gr_max;
  int n = P.n_ocp;
  if (s < P.ocp_soc[0] || s > P.ocp_soc[n - 1]) return 0.0;
  int lo = 0, hi = n;   // k = number of knots <= s (searchsorted side=right)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (P.ocp_soc[mid] <= s) lo = mid + 1; else hi = mid;
  }
  int seg = lo - 1;
  if (seg < 0) seg = 0;
  if (seg > n - 2) seg = n - 2;
  return (P.ocp_v[seg + 1] - P.ocp_v[seg]) / (P.ocp_soc[seg + 1] - P.ocp_soc[seg]) / P.c_gr_max;
}

// f_pre and its derivative (echem/kinetics.py:71-87).
__device__ __host__ inline double f_pre_dev(double n, double nc) {
  double n4 = (n * n) * (n * n);
  double nc4 = (nc * nc) * (nc * nc);
  return n4 / (nc4 + n4);
}
__device__ __host__ inline double f_pre_deriv_dev(double n, double nc) {
  double nc4 = (nc * nc) * (nc * nc);
  double d = nc4 + (n * n) * (n * n);
  return 4.0 * (n * n * n) * nc4 / (d * d);
}

// Stripping current with the implicit-inventory regularization
// (operator.py:271-320).  Returns i; optionally the two Jacobian entries.
__device__ __host__ inline double strip_current_dev(double c_el, double phi_pl, double phi_el,
                                                    double n_face, double beta, const DevParams& P,
                                                    double* di_dce, double* di_dpp) {
  double vt = P.vt;
  double arg = (phi_pl - phi_el) / vt;
  double ex = exp(arg), emx = exp(-arg);
  double E = P.i00_plel * sqrt(c_el);
  if (beta == 0.0) {
    double fp = f_pre_dev(n_face, P.n_const);
    double i = E * (fp * ex - emx);
    if (di_dce) {
      *di_dce = 0.5 * i / c_el;
      *di_dpp = E * (fp * ex + emx) / vt;
    }
    return i;
  }
  double lo = -E * emx, hi = E * (ex - emx);
  double fp0 = f_pre_dev(n_face, P.n_const);
  double i = fmin(fmax(E * (fp0 * ex - emx), lo), hi);
  for (int it = 0; it < 60; ++it) {
    double n_end = fmax(n_face - beta * i, 0.0);
    double f = f_pre_dev(n_end, P.n_const);
    double fd = n_end > 0.0 ? f_pre_deriv_dev(n_end, P.n_const) : 0.0;
    double g = i - E * (f * ex - emx);
    double gi = 1.0 + E * ex * fd * beta;
    double i_new = fmin(fmax(i - g / gi, lo), hi);
    bool done = fabs(i_new - i) <= 1e-14 * (1.0 + fabs(i_new));
    i = i_new;
    if (done) break;
  }
  if (di_dce) {
    double n_end = fmax(n_face - beta * i, 0.0);
    double f = f_pre_dev(n_end, P.n_const);
    double fd = n_end > 0.0 ? f_pre_deriv_dev(n_end, P.n_const) : 0.0;
    double gi = 1.0 + E * ex * fd * beta;
    *di_dce = (0.5 / c_el) * E * (f * ex - emx) / gi;
    *di_dpp = E * (f * ex + emx) / vt / gi;
  }
  return i;
}

// Interface face record kinds in the compacted list.
enum : int8_t { IF_BV = 0, IF_CE = 1, IF_STRIP = 2 };

// Device buffer RAII.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) HC_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
};

struct Amg;   // hc_amg.cu
struct Work;  // hc_solver.cu
struct KrylovGraphs;  // hc_krylov.cu
struct TmaCache;      // hc_tma.cuh
struct NewtonGraph;   // hc_solver.cu
void destroy_newton_graph(NewtonGraph* g);
void destroy_krylov_graphs(KrylovGraphs* g);

// The device-resident operator: geometry, DOF numbering, compacted face lists
// and the work space of the implicit step.
struct Operator {
  DevParams P;
  hc_params host_params;
  double voxel_um = 1.0;
  hc_info info;
  int n_sm = 148;

  DBuf<uint8_t> labels;        // [nvox]
  DBuf<int32_t> lab4;          // labels widened to 32 bit (cp.async staging)
  DBuf<int32_t> labt;          // TMA face word (hc_tma.cuh), 0 = outside
  DBuf<int2> if_fslot;         // TMA stencil: per interface face, its slot on the solid / electrolyte side
  TmaCache* tma = nullptr;     // tensor maps of the TMA stencils
  DBuf<int32_t> cdof, pdof;    // [nvox], -1 where absent
  DBuf<int32_t> c_vox, p_vox;  // packed index -> voxel
  DBuf<int32_t> plated_vox;    // [n_plated] ascending
  // interface faces, reference order within each family; unified SoA list
  // (bv first, then ce, then strip) for the kernels
  DBuf<int32_t> if_solid, if_el, if_slot;  // slot: plated slot for strip, -1 else
  DBuf<int8_t> if_kind;
  int64_t n_if = 0;
  DBuf<int32_t> elel_lo, elel_hi;          // only materialised for export
  DBuf<int32_t> if_rank;                   // [nvox] rank among interface voxels or -1
  DBuf<int32_t> if_dir;                    // [6 * n_if_vox] face id per direction or -1

  // grid-layout work space (double2 = (c, phi) per voxel)
  DBuf<double2> xg, xg2, vg, outg;
  DBuf<double> cprev;          // c_prev * inv_dt per voxel (time term)
  DBuf<double> npl;            // plated inventory per slot
  DBuf<double> if_coef;        // 3 x n_if Jacobian coefficients (linearized)
  DBuf<double> if_vcoef;       // the same per interface voxel and direction: [3][6 n_if_vox]
  DBuf<double> if_cslot;       // TMA stencil: (alpha, beta, gamma) per interface face slot
  DBuf<int2> elz;              // TMA stencil: electrolyte z range per 32 x 8 tile column
  DBuf<double> if_islot;       // TMA residual: interface current per face slot
  DBuf<double> if_cur;         // cp.async residual: interface current per face
  DBuf<int32_t> tp_off;        // TMA stencil: first slot per (tile, plane), slots tile-plane ordered
  int2 cz = {0, 0};            // planes [cz.x, cz.y) hold every c row (electrolyte / graphite voxels)
  DBuf<double> inv_c;          // gX / c per electrolyte voxel (linearized)
  DBuf<double> red;            // reduction scratch
  DBuf<double> host_x, host_npl;  // staging for the host-buffer entry point
  Amg* amg = nullptr;
  Work* work = nullptr;
  int krylov_log = 0;
  int stencil_kind = 3;            // 2: cp.async ring, 3: TMA ring (nx % 4 == 0, else 2)
  bool dev_krylov = true;          // device-resident BiCGStab (hc_krylov.cu)
  int krylov_batch = 4;            // iteration graphs launched per status check (fallback)
  bool krylov_while = true;        // whole solve as one graph with a device-side WHILE node
  // whole Newton solve as one graph (conditional nodes): no host sync per Newton iteration;
  // measured at parity with the host-controlled loop at the exact Krylov tolerance (large
  // cell 88.2 vs 87.8 ms/step, medium 20.2 vs 20.3); HC_NEWTON_DEV=0 selects the host loop
  bool newton_dev = true;
  NewtonGraph* ng = nullptr;
  bool capturing = false;          // inside a stream capture (no nested capture)
  KrylovGraphs* kg = nullptr;
  cudaStream_t stream = nullptr;   // private non-blocking stream (graph capture needs one)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // Newton trace of newton_solve (its iterates and residual norms, newton.py:153-161)
  // and its optional source term (newton.py:107-108).  While any of these is set the
  // host-controlled Newton loop runs (the device graph records neither).
  double* iter_out = nullptr;      // packed iterates [iter_max][n_total] (device) or null
  int iter_max = 0, iter_count = 0;
  bool trace_norms = false;
  std::vector<double> norm_log;    // |F| of the guess and of every accepted iterate
  const double2* src = nullptr;    // grid-layout source added to every residual, or null
  // set when the last Newton failure was a Krylov failure on a preconditioner that was
  // not rebuilt in that solve: the caller rebuilds it and retries at the same dt
  bool krylov_fail_stale = false;

  ~Operator();
};

// kernels / helpers implemented in hc_operator.cu
void scatter_packed(const Operator& op, const double* x, double2* xg, bool c_fill_one,
                    cudaStream_t s);
void gather_packed(const Operator& op, const double2* xg, double* x, cudaStream_t s);
// residual in grid layout: parts bitmask
enum : int { PART_LIN = 1, PART_BV = 2, PART_1C = 4, PART_BND = 8, PART_TIME = 16 };
// scalar-mode stencil flag: write the output with stride 2, i.e. into one component of a
// double2 (c, phi) vector (the preconditioner's final sweeps fill z directly)
constexpr int FL_OSTRIDE2 = 1 << 16;
void residual_grid(Operator& op, const double2* xg, const double* npl, double mu, double beta,
                   int parts, const double* cprev_scaled, double inv_dt, double2* out,
                   cudaStream_t s, int which = 3);  // which: 1 stencil kernel, 2 interface kernel
void linearize(Operator& op, const double2* xg, const double* npl, double beta, cudaStream_t s);
// stripping current per stripping face (operator.py:391-399) into out[n_strip]
void strip_currents(Operator& op, const double2* xg, const double* npl, double beta, double* out,
                    cudaStream_t s);
// J v with the linearization stored in op.  flags: 1 add mass (inv_dt on c rows),
// 2 row transform T (electrolyte c row -= t+ phi row), 4 include 1/c terms,
// 8 phi rows only (c rows written as 0)
void jvp_grid(Operator& op, const double2* vg, double inv_dt, int flags, double2* out,
              cudaStream_t s, int which = 3);
int jvp_grid_dot(Operator& op, const double2* vg, double inv_dt, int flags, double2* out,
                 const double2* a, double* part, int two, cudaStream_t s);
double norm2_grid(Operator& op, const double2* v, int field_mask, cudaStream_t s);
Operator* create_operator(const uint8_t* labels_host, int nx, int ny, int nz, double voxel_um,
                          const hc_params& hp);
// new material parameters on the same geometry (DevParams, info); the caller drops the caches
void set_params(Operator& op, const hc_params& hp);

}  // namespace hc

namespace hc {
// ---- programmatic dependent launch (PDL) --------------------------------------------
// Kernels of the Krylov / multigrid loop are launched with programmatic stream
// serialization, so a kernel's launch and prologue overlap its predecessor's tail.
// Every such kernel calls pdl_wait() as its first statement (before any early exit):
// it blocks until the predecessor grid has completed and its writes are visible, which
// also keeps the ordering transitive along the stream.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the successor grid launch now (its CTAs then wait in pdl_wait) when this grid is
// at most about one wave, so an early launch cannot steal slots from our own later waves.
__device__ __forceinline__ void pdl_trigger_small() {
  if (gridDim.x * gridDim.y * gridDim.z <= 592u) asm volatile("griddepcontrol.launch_dependents;");
}

bool pdl_enabled();   // HC_PDL (default 1)

template <typename... KArgs, typename... Args>
inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  HC_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}
}  // namespace hc
