// Operator setup (dofmap + face classification/compaction), residual, Jacobian
// linearization and matrix-free Jacobian-vector product on the voxel grid.
//
// Reference: fvm/dofmap.py:71-101 (numbering, validation), fvm/operator.py:121-242
// (face classification, face lists), operator.py:246-389 (residual),
// operator.py:402-471 (analytic Jacobian).
//
// Grid layout: one double2 (c, phi) per voxel, x fastest.  Absent DOFs hold
// c = 1 (never read) and phi = 0 (the grounded value).
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "hc_internal.cuh"
#include "hc_stencil.cuh"
#include "hc_tma.cuh"
#include <cudaTypedefs.h>

namespace hc {

namespace {

constexpr int TPB = 256;

inline int blocks_for(long long n, int tpb = TPB) { return (int)((n + tpb - 1) / tpb); }

__device__ __forceinline__ void coords(const DevParams& P, long long v, int& x, int& y, int& z) {
  x = (int)(v % P.nx);
  long long t = v / P.nx;
  y = (int)(t % P.ny);
  z = (int)(t / P.ny);
}

__device__ __forceinline__ bool grounded(const DevParams& P, uint8_t lab, int z) {
  return z == P.nz - 1 && lab == CC;
}

// face f in reference enumeration order -> (lo, hi) voxel (operator.py:132-138)
__device__ __forceinline__ void face_voxels(const DevParams& P, long long f, long long& lo,
                                            long long& hi) {
  long long nx = P.nx, ny = P.ny, nz = P.nz;
  long long fz = (nz - 1) * ny * nx, fy = nz * (ny - 1) * nx;
  if (f < fz) {
    lo = f;
    hi = f + ny * nx;
  } else if (f < fz + fy) {
    long long g = f - fz;
    long long x = g % nx, t = g / nx, y = t % (ny - 1), z = t / (ny - 1);
    lo = (z * ny + y) * nx + x;
    hi = lo + nx;
  } else {
    long long g = f - fz - fy;
    long long x = g % (nx - 1), t = g / (nx - 1), y = t % ny, z = t / ny;
    lo = (z * ny + y) * nx + x;
    hi = lo + 1;
  }
}

// ---------------------------------------------------------------- setup kernels
__global__ void k_masks(DevParams P, const uint8_t* __restrict__ lab, int32_t* cmask,
                        int32_t* pmask, int32_t* plmask) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  uint8_t a = lab[v];
  int z = (int)(v / P.nxy);
  cmask[v] = (a == GR || a == EL) ? 1 : 0;
  pmask[v] = grounded(P, a, z) ? 0 : 1;
  plmask[v] = (a == PL) ? 1 : 0;
}

__global__ void k_finalize_numbering(long long n, const int32_t* __restrict__ mask,
                                     int32_t* __restrict__ num, int32_t* __restrict__ inv) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (mask[v]) {
    int32_t k = num[v];
    if (inv) inv[k] = (int32_t)v;
  } else {
    num[v] = -1;
  }
}

// per-face kind code with error flags: bit 0 forbidden, bit 1 kinetics on grounded face
__global__ void k_face_check(DevParams P, const uint8_t* __restrict__ lab, long long n_faces,
                             int* __restrict__ err, unsigned long long* __restrict__ first_bad) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_faces) return;
  long long lo, hi;
  face_voxels(P, f, lo, hi);
  uint8_t a = lab[lo], b = lab[hi];
  uint8_t k = kind_of(a, b);
  bool glo = grounded(P, a, (int)(lo / P.nxy)), ghi = grounded(P, b, (int)(hi / P.nxy));
  if (k == K_FORBID && !(glo && ghi)) {
    atomicOr(err, 1);
    atomicMin(first_bad, (unsigned long long)f);
  }
  if ((glo != ghi) && (k == K_BV || k == K_CE || k == K_STRIP)) atomicOr(err, 2);
}

struct FaceIsKind {
  DevParams P;
  const uint8_t* lab;
  uint8_t kind;
  __device__ bool operator()(const long long& f) const {
    long long lo, hi;
    face_voxels(P, f, lo, hi);
    uint8_t a = lab[lo], b = lab[hi];
    if (kind == 7) {
      if (kind_of(a, b) != K_CONT || a != EL) return false;
    } else if (kind_of(a, b) != kind) {
      return false;
    }
    bool glo = grounded(P, a, (int)(lo / P.nxy)), ghi = grounded(P, b, (int)(hi / P.nxy));
    return !glo && !ghi;
  }
};

// interface faces oriented solid first (operator.py:204-208)
__global__ void k_orient(DevParams P, const uint8_t* __restrict__ lab,
                         const long long* __restrict__ faces, long long n, int8_t kind,
                         const int32_t* __restrict__ plslot, int32_t* solid, int32_t* el,
                         int32_t* slot, int8_t* kinds) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long lo, hi;
  face_voxels(P, faces[i], lo, hi);
  bool a_is_el = lab[lo] == EL;
  long long so = a_is_el ? hi : lo, e = a_is_el ? lo : hi;
  solid[i] = (int32_t)so;
  el[i] = (int32_t)e;
  slot[i] = kind == IF_STRIP ? plslot[so] : -1;
  kinds[i] = kind;
}

__global__ void k_elel_pairs(DevParams P, const long long* __restrict__ faces, long long n,
                             int32_t* lo_out, int32_t* hi_out) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long lo, hi;
  face_voxels(P, faces[i], lo, hi);
  lo_out[i] = (int32_t)lo;
  hi_out[i] = (int32_t)hi;
}

// per-voxel interface map: mark voxels incident to interface faces
__global__ void k_if_mark(long long n_if, const int32_t* __restrict__ so,
                          const int32_t* __restrict__ el, int32_t* mark) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  mark[so[f]] = 1;
  mark[el[f]] = 1;
}

__device__ __forceinline__ int dir_to(const DevParams& P, long long a, long long b) {
  long long za = a / P.nxy, zb = b / P.nxy;
  if (za != zb) return zb > za ? 5 : 4;
  long long ya = (a / P.nx) % P.ny, yb = (b / P.nx) % P.ny;
  if (ya != yb) return yb > ya ? 3 : 2;
  return b > a ? 1 : 0;
}

__global__ void k_if_dirs(DevParams P, long long n_if, const int32_t* __restrict__ so,
                          const int32_t* __restrict__ el, const int32_t* __restrict__ rank,
                          int32_t* __restrict__ dirs) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  int32_t s = so[f], e = el[f];
  dirs[6LL * rank[s] + dir_to(P, s, e)] = (int32_t)f;
  dirs[6LL * rank[e] + dir_to(P, e, s)] = (int32_t)f;
}

// ---- electrolyte connectivity (dofmap.py:57-68): union-find on the device ----
__device__ int32_t uf_find(int32_t* par, int32_t v) {
  while (true) {
    int32_t p = par[v];
    if (p == v) return v;
    int32_t gp = par[p];
    if (gp != p) par[v] = gp;  // path halving (benign race)
    v = p;
  }
}

__device__ void uf_union(int32_t* par, int32_t a, int32_t b) {
  while (true) {
    a = uf_find(par, a);
    b = uf_find(par, b);
    if (a == b) return;
    if (a < b) { int32_t t = a; a = b; b = t; }
    // hook larger root a under b
    int32_t old = atomicCAS(&par[a], a, b);
    if (old == a) return;
    a = old;
  }
}

__global__ void k_uf_init(DevParams P, const uint8_t* __restrict__ lab, int32_t* par) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  par[v] = (int32_t)v;
}

__global__ void k_uf_merge(DevParams P, const uint8_t* __restrict__ lab, int32_t* par) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  if (lab[v] != EL) return;
  int x, y, z;
  coords(P, v, x, y, z);
  if (x + 1 < P.nx && lab[v + 1] == EL) uf_union(par, (int32_t)v, (int32_t)(v + 1));
  if (y + 1 < P.ny && lab[v + P.nx] == EL) uf_union(par, (int32_t)v, (int32_t)(v + P.nx));
  if (z + 1 < P.nz && lab[v + P.nxy] == EL) uf_union(par, (int32_t)v, (int32_t)(v + P.nxy));
}

__global__ void k_uf_touch(DevParams P, const uint8_t* __restrict__ lab, int32_t* par,
                           uint8_t* touch) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  if (lab[v] != EL) return;
  int x, y, z;
  coords(P, v, x, y, z);
  uint8_t m = 0;
  auto chk = [&](long long nb) {
    uint8_t b = lab[nb];
    if (b == GR) m |= 1;
    if (b == FOIL) m |= 2;
  };
  if (x > 0) chk(v - 1);
  if (x + 1 < P.nx) chk(v + 1);
  if (y > 0) chk(v - P.nx);
  if (y + 1 < P.ny) chk(v + P.nx);
  if (z > 0) chk(v - P.nxy);
  if (z + 1 < P.nz) chk(v + P.nxy);
  if (m) {
    int32_t r = uf_find(par, (int32_t)v);
    atomicOr((unsigned int*)&touch[r & ~3], (unsigned int)m << (8 * (r & 3)));
  }
}

__global__ void k_uf_both(long long n, const uint8_t* __restrict__ touch, int* ok) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= n) return;
  if (touch[v] == 3) *ok = 1;
}

// --------------------------------------------------------------- layout kernels
__global__ void k_scatter(DevParams P, int n_c, int n_p, const int32_t* __restrict__ c_vox,
                          const int32_t* __restrict__ p_vox, const double* __restrict__ x,
                          double2* __restrict__ xg) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n_c) xg[c_vox[i]].x = x[i];
  if (i < n_p) xg[p_vox[i]].y = x[n_c + i];
}

__global__ void k_fill(long long n, double2* xg, double c, double p) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v < n) xg[v] = make_double2(c, p);
}

__global__ void k_gather(int n_c, int n_p, const int32_t* __restrict__ c_vox,
                         const int32_t* __restrict__ p_vox, const double2* __restrict__ xg,
                         double* __restrict__ x) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n_c) x[i] = xg[c_vox[i]].x;
  if (i < n_p) x[n_c + i] = xg[p_vox[i]].y;
}

// Interface currents over the compacted face list (operator.py:331-357), cp.async stencil
// path (grids without tensor-map tiles): one current per face ...
__global__ void __launch_bounds__(TPB) k_residual_iface(
    DevParams P, long long n_if, const int32_t* __restrict__ so, const int32_t* __restrict__ el,
    const int32_t* __restrict__ slot, const int8_t* __restrict__ kind,
    const double2* __restrict__ X, const double* __restrict__ npl, double beta,
    double* __restrict__ cur) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  int32_t s = so[f], e = el[f];
  double2 xs = X[s], xe = X[e];
  int8_t k = kind[f];
  double i;
  if (k == IF_BV) {
    double eta = xs.y - ocp_dev(xs.x, P) - xe.y;
    double root = sqrt(xs.x * xe.x);
    i = 2.0 * P.i00_grel * root * sinh(eta / P.vt);
  } else if (k == IF_CE) {
    i = 2.0 * P.i00_ceel * sinh((xs.y - xe.y) / P.vt);
  } else {
    i = strip_current_dev(xe.x, xs.y, xe.y, npl[slot[f]], beta, P, nullptr, nullptr);
  }
  cur[f] = P.sc * i;
}
// ... gathered per interface voxel over its faces in direction order (fixed order, no
// floating-point atomics): the solid row takes +i (its c row only on BV faces), the
// electrolyte row -i on both equations
__global__ void __launch_bounds__(TPB) k_residual_iface_gather(
    long long nvox, const int32_t* __restrict__ rank, const int32_t* __restrict__ dirs,
    const int32_t* __restrict__ so, const int8_t* __restrict__ kind, const double* __restrict__ cur,
    double2* __restrict__ out) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= nvox) return;
  const int rk = rank[v];
  if (rk < 0) return;
  double dc = 0.0, dp = 0.0;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int f = dirs[6LL * rk + d];
    if (f < 0) continue;
    const double q = cur[f];
    if (so[f] == (int32_t)v) {
      if (kind[f] == IF_BV) dc += q;
      dp += q;
    } else {
      dc -= q;
      dp -= q;
    }
  }
  double2 o = out[v];
  o.x += dc;
  o.y += dp;
  out[v] = o;
}

// The same currents written once per face slot, oriented from each side's row (solid
// +i, electrolyte -i), for the TMA residual stencil to gather: no atomics.
__global__ void __launch_bounds__(TPB) k_residual_islot(
    DevParams P, long long n_if, const int32_t* __restrict__ so, const int32_t* __restrict__ el,
    const int32_t* __restrict__ slot, const int8_t* __restrict__ kind, const int2* __restrict__ fslot,
    const double2* __restrict__ X, const double* __restrict__ npl, double beta,
    double* __restrict__ islot) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  int32_t s = so[f], e = el[f];
  double2 xs = X[s], xe = X[e];
  int8_t k = kind[f];
  double i;
  if (k == IF_BV) {
    double eta = xs.y - ocp_dev(xs.x, P) - xe.y;
    double root = sqrt(xs.x * xe.x);
    i = 2.0 * P.i00_grel * root * sinh(eta / P.vt);
  } else if (k == IF_CE) {
    i = 2.0 * P.i00_ceel * sinh((xs.y - xe.y) / P.vt);
  } else {
    i = strip_current_dev(xe.x, xs.y, xe.y, npl[slot[f]], beta, P, nullptr, nullptr);
  }
  const double q = P.sc * i;
  const int2 fs = fslot[f];
  islot[fs.x] = q;
  islot[fs.y] = -q;
}

// Stripping current of every stripping face (operator.py:391-399), faces f0.. of the
// unified list (bv | ce | strip), unscaled A/m^2.
__global__ void k_strip_currents(DevParams P, long long f0, long long n, const int32_t* __restrict__ so,
                                 const int32_t* __restrict__ el, const int32_t* __restrict__ slot,
                                 const double2* __restrict__ X, const double* __restrict__ npl, double beta,
                                 double* __restrict__ out) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const long long f = f0 + k;
  const double2 xs = X[so[f]], xe = X[el[f]];
  out[k] = strip_current_dev(xe.x, xs.y, xe.y, npl[slot[f]], beta, P, nullptr, nullptr);
}

// --------------------------------------------------------------- linearization
__global__ void k_lin_iface(DevParams P, long long n_if, const int32_t* __restrict__ so,
                            const int32_t* __restrict__ el, const int32_t* __restrict__ slot,
                            const int8_t* __restrict__ kind, const double2* __restrict__ X,
                            const double* __restrict__ npl, double beta,
                            double* __restrict__ coef) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  int32_t s = so[f], e = el[f];
  double2 xs = X[s], xe = X[e];
  int8_t k = kind[f];
  double a = 0.0, b = 0.0, g = 0.0;
  if (k == IF_BV) {
    double cg = xs.x, ce = xe.x;
    double eta = xs.y - ocp_dev(cg, P) - xe.y;
    double root = sqrt(cg * ce);
    double sh = sinh(eta / P.vt), ch = cosh(eta / P.vt);
    a = 2.0 * P.i00_grel * (0.5 * sqrt(ce / cg) * sh - root * ch * ocp_slope_dev(cg, P) / P.vt);
    b = P.i00_grel * sqrt(cg / ce) * sh;
    g = 2.0 * P.i00_grel * root * ch / P.vt;
  } else if (k == IF_CE) {
    g = 2.0 * P.i00_ceel * cosh((xs.y - xe.y) / P.vt) / P.vt;
  } else {
    strip_current_dev(xe.x, xs.y, xe.y, npl[slot[f]], beta, P, &b, &g);
  }
  coef[f] = P.sc * a;
  coef[n_if + f] = P.sc * b;
  coef[2 * n_if + f] = P.sc * g;
}

// per interface voxel and direction: the face's three coefficients oriented from that
// voxel's row (layout [3][6 * n_if_vox]) so the stencil kernels read them with one load
__global__ void k_lin_scatter(DevParams P, long long n_if, const int32_t* __restrict__ so,
                              const int32_t* __restrict__ el, const int32_t* __restrict__ rank,
                              const double* __restrict__ coef, long long nslot,
                              double* __restrict__ ifv) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  const int s = so[f], e = el[f];
  const double ca = coef[f], cb = coef[n_if + f], cg = coef[2 * n_if + f];
  const long long is = 6LL * rank[s] + dir_to(P, s, e), ie = 6LL * rank[e] + dir_to(P, e, s);
  // row-oriented: the face adds alpha c_row + beta c_nbr + gamma (phi_row - phi_nbr) to the
  // row's phi equation (solid: +i, electrolyte: -i; ca is zero except on BV faces)
  ifv[is] = ca; ifv[nslot + is] = cb; ifv[2 * nslot + is] = cg;
  ifv[ie] = -cb; ifv[nslot + ie] = -ca; ifv[2 * nslot + ie] = cg;
}

// the same, into the compact per-face slots of the TMA stencil (AoS, 32 B per slot: the
// triple + pad; a voxel's slots are consecutive in direction order, first slot in its
// label word)
__global__ void k_lin_scatter_c(DevParams P, long long n_if, const int32_t* __restrict__ so,
                                const int32_t* __restrict__ el, const int2* __restrict__ fslot,
                                const double* __restrict__ coef, double* __restrict__ cs) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= n_if) return;
  const int s = so[f], e = el[f];
  const double ca = coef[f], cb = coef[n_if + f], cg = coef[2 * n_if + f];
  const int2 fs = fslot[f];
  const long long is = 4LL * fs.x, ie = 4LL * fs.y;
  cs[is] = ca; cs[is + 1] = cb; cs[is + 2] = cg;
  cs[ie] = -cb; cs[ie + 1] = -ca; cs[ie + 2] = cg;
}

__global__ void k_lin_invc(DevParams P, const uint8_t* __restrict__ lab,
                           const double2* __restrict__ X, double* __restrict__ w) {
  long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (v >= P.nvox) return;
  w[v] = lab[v] == EL ? P.gX / X[v].x : 0.0;
}

// ------------------------------------------------------------------ reductions
// per-block partial sums of squares of the selected fields; field_mask 1 = c, 2 = phi
__global__ void k_sumsq(long long n, const double2* __restrict__ v, int field_mask,
                        double* __restrict__ part) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 a = v[i];
    if (field_mask & 1) acc += a.x * a.x;
    if (field_mask & 2) acc += a.y * a.y;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

}  // namespace

// ================================================================ host wrappers
void scatter_packed(const Operator& op, const double* x, double2* xg, bool c_fill_one,
                    cudaStream_t s) {
  long long nv = op.P.nvox;
  k_fill<<<blocks_for(nv), TPB, 0, s>>>(nv, xg, c_fill_one ? 1.0 : 0.0, 0.0); HC_COUNT();
  long long n = std::max(op.info.n_c, op.info.n_p);
  if (n) k_scatter<<<blocks_for(n), TPB, 0, s>>>(op.P, (int)op.info.n_c, (int)op.info.n_p,
                                                 op.c_vox.p, op.p_vox.p, x, xg); HC_COUNT();
  HC_CHECK_LAUNCH();
}

void gather_packed(const Operator& op, const double2* xg, double* x, cudaStream_t s) {
  long long n = std::max(op.info.n_c, op.info.n_p);
  if (n) k_gather<<<blocks_for(n), TPB, 0, s>>>((int)op.info.n_c, (int)op.info.n_p, op.c_vox.p,
                                                op.p_vox.p, xg, x); HC_COUNT();
  HC_CHECK_LAUNCH();
}

void residual_grid(Operator& op, const double2* xg, const double* npl, double mu, double beta,
                   int parts, const double* cprev, double inv_dt, double2* out, cudaStream_t s,
                   int which) {
  if (op.tma && op.stencil_kind == 3) {
    // deterministic: face currents into per-slot storage, gathered by the stencil
    if ((which & 2) && (parts & PART_BV) && op.n_if)
      k_residual_islot<<<blocks_for(op.n_if), TPB, 0, s>>>(op.P, op.n_if, op.if_solid.p, op.if_el.p,
                                                           op.if_slot.p, op.if_kind.p, op.if_fslot.p, xg,
                                                           npl, beta, op.if_islot.p); HC_COUNT();
    if ((which & 1) && res_launch_tma(op, xg, mu, parts, cprev, inv_dt, out, s)) {
      HC_COUNT();
      HC_CHECK_LAUNCH();
      return;
    }
    if (which & 1) throw Error(HC_ERR_CUDA, "TMA residual launch failed");
    HC_CHECK_LAUNCH();
    return;
  }
  if (which & 1) {
    res_launch_p(op.P, op.lab4.p, xg, mu, parts, cprev, inv_dt, out, op.n_sm, s);
    HC_COUNT();
  }
  if ((which & 2) && (parts & PART_BV) && op.n_if) {
    k_residual_iface<<<blocks_for(op.n_if), TPB, 0, s>>>(op.P, op.n_if, op.if_solid.p,
                                                         op.if_el.p, op.if_slot.p, op.if_kind.p,
                                                         xg, npl, beta, op.if_cur.p); HC_COUNT();
    k_residual_iface_gather<<<blocks_for(op.P.nvox), TPB, 0, s>>>(op.P.nvox, op.if_rank.p, op.if_dir.p,
                                                                  op.if_solid.p, op.if_kind.p,
                                                                  op.if_cur.p, out); HC_COUNT();
  }
  HC_CHECK_LAUNCH();
}

void strip_currents(Operator& op, const double2* xg, const double* npl, double beta, double* out,
                    cudaStream_t s) {
  const long long n = op.info.n_strip;
  if (!n) return;
  k_strip_currents<<<blocks_for(n), TPB, 0, s>>>(op.P, op.info.n_bv + op.info.n_ce, n, op.if_solid.p,
                                                 op.if_el.p, op.if_slot.p, xg, npl, beta, out); HC_COUNT();
  HC_CHECK_LAUNCH();
}

void linearize(Operator& op, const double2* xg, const double* npl, double beta, cudaStream_t s) {
  if (op.n_if) {
    k_lin_iface<<<blocks_for(op.n_if), TPB, 0, s>>>(op.P, op.n_if, op.if_solid.p, op.if_el.p,
                                                    op.if_slot.p, op.if_kind.p, xg, npl, beta,
                                                    op.if_coef.p); HC_COUNT();
    if (op.tma)
      k_lin_scatter_c<<<blocks_for(op.n_if), TPB, 0, s>>>(op.P, op.n_if, op.if_solid.p, op.if_el.p,
                                                          op.if_fslot.p, op.if_coef.p, op.if_cslot.p); HC_COUNT();
    long long nslot = (long long)op.if_dir.n;
    k_lin_scatter<<<blocks_for(op.n_if), TPB, 0, s>>>(op.P, op.n_if, op.if_solid.p, op.if_el.p,
                                                      op.if_rank.p, op.if_coef.p, nslot,
                                                      op.if_vcoef.p); HC_COUNT();
  }
  k_lin_invc<<<blocks_for(op.P.nvox), TPB, 0, s>>>(op.P, op.labels.p, xg, op.inv_c.p); HC_COUNT();
  HC_CHECK_LAUNCH();
}

bool tma_encode(CUtensorMap* m, const void* ptr, int kind, int nx, int ny, int nz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn || !ptr || (reinterpret_cast<uintptr_t>(ptr) & 15)) return false;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], es[3] = {1, 1, 1};
  CUtensorMapDataType dt;
  size_t ebytes;
  if (kind == 0) {         // int32 labels, 40-wide boxes (160 B rows)
    dt = CU_TENSOR_MAP_DATA_TYPE_INT32; ebytes = 4; dims[0] = nx; box[0] = T_LW;
  } else if (kind == 1) {  // double2 as pairs of float64
    dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; ebytes = 8; dims[0] = 2 * (cuuint64_t)nx; box[0] = 2 * T_QW;
  } else {                 // double
    dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64; ebytes = 8; dims[0] = nx; box[0] = T_DW;
  }
  dims[1] = ny; dims[2] = nz;
  box[1] = T_TH; box[2] = 1;
  strides[0] = dims[0] * ebytes;
  strides[1] = strides[0] * ny;
  if (strides[0] % 16) return false;
  CUresult r = fn(m, dt, 3, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void jvp_grid(Operator& op, const double2* vg, double inv_dt, int flags, double2* out,
              cudaStream_t s, int which) {
  if (which & 1) {
    FineArgs F{op.labels.p, op.if_rank.p, op.if_vcoef.p, (long long)op.if_dir.n, op.inv_c.p,
               op.if_cslot.p, op.elz.p, nullptr, op.tp_off.p};
    fine_launch_op<SM_FULL, EP_STORE>(op, F, vg, nullptr, nullptr, nullptr, 0.0, inv_dt, flags, out,
                                      nullptr, s);
    HC_COUNT();
  }
  HC_CHECK_LAUNCH();
}

// J v through the TMA stencil with the per-CTA partial dot products out.a (and out.out
// when two) fused into its epilogue; returns the number of partials, 0 if the TMA path is
// not available (nothing launched then)
int jvp_grid_dot(Operator& op, const double2* vg, double inv_dt, int flags, double2* out,
                 const double2* a, double* part, int two, cudaStream_t s) {
  if (op.stencil_kind != 3 || !op.tma) return 0;
  int nblk = 0;
  FineArgs F{op.labels.p, op.if_rank.p, op.if_vcoef.p, (long long)op.if_dir.n, op.inv_c.p,
             op.if_cslot.p, op.elz.p, nullptr, op.tp_off.p, a, part, two, &nblk};
  if (!fine_launch_tma<SM_FULL, EP_STORE>(*op.tma, op.P, F, op.labt.p, vg, nullptr, nullptr, nullptr, 0.0,
                                          inv_dt, flags, out, nullptr, op.n_sm, s))
    return 0;
  HC_COUNT();
  HC_CHECK_LAUNCH();
  return nblk;
}

double norm2_grid(Operator& op, const double2* v, int field_mask, cudaStream_t s) {
  int nb = std::min<long long>(blocks_for(op.P.nvox), 4 * op.n_sm);
  k_sumsq<<<nb, TPB, 0, s>>>(op.P.nvox, v, field_mask, op.red.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  std::vector<double> h(nb);
  HC_CUDA(cudaMemcpyAsync(h.data(), op.red.p, nb * sizeof(double), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  double acc = 0.0;
  for (double d : h) acc += d;
  return std::sqrt(acc);
}

// ================================================================ construction
static DevParams make_dev_params(const hc_params& hp, int nx, int ny, int nz, double voxel_um) {
  DevParams P;
  std::memset(&P, 0, sizeof(P));
  P.nx = nx;
  P.ny = ny;
  P.nz = nz;
  P.nxy = (long long)nx * ny;
  P.nvox = P.nxy * nz;
  const double F = hp.faraday, R = hp.gas_constant, h = voxel_um * 1e-6;
  P.h = h;
  P.gF2 = 1.0 / (F * h * h);
  P.sc = 1.0 / (F * h);
  P.inv_h2 = 1.0 / (h * h);
  P.d_gr = hp.d_gr;
  P.d_el = hp.d_el;
  P.t_plus = hp.t_plus;
  P.kappa = hp.kappa_el;
  P.sigma_gr = hp.sigma_gr;
  P.sig[EL] = hp.kappa_el;
  P.sig[GR] = hp.sigma_gr;
  P.sig[PL] = hp.sigma_pl;
  P.sig[FOIL] = hp.sigma_li;
  P.sig[CW] = hp.sigma_cc;
  P.sig[CC] = hp.sigma_cc;
  P.gX = (hp.kappa_el * (hp.t_plus - 1.0) * R * hp.temperature * (1.0 + hp.dlnf_dlnc)) /
         (F * F * h * h);
  P.vt = 2.0 * R * hp.temperature / F;
  P.i00_grel = hp.i00_grel;
  P.i00_ceel = hp.i00_ceel;
  P.i00_plel = hp.i00_plel;
  P.c_gr_max = hp.c_gr_max;
  P.n_const = hp.c_li_metal * hp.n_const_thickness * (h * h);
  P.drive = -1.0 / (F * h);
  P.n_ocp = hp.n_ocp;
  for (int k = 0; k < hp.n_ocp; ++k) {
    P.ocp_soc[k] = hp.ocp_soc[k];
    P.ocp_v[k] = hp.ocp_v[k];
  }
  for (int a = 0; a < N_PHASES; ++a)
    for (int b = 0; b < N_PHASES; ++b) {
      int i = a * N_PHASES + b;
      uint8_t k = kind_of((uint8_t)a, (uint8_t)b);
      P.gP[i] = P.gC[i] = P.gMig[i] = 0.0;
      P.ifc[i] = (k == K_BV || k == K_CE || k == K_STRIP) ? 1 : 0;
      if (k == K_CONT) {
        P.gP[i] = (a == GR ? P.sigma_gr : (a == EL ? P.kappa : P.sig[a])) * P.gF2;
        if (a == GR) P.gC[i] = P.d_gr * P.inv_h2;
        if (a == EL) {
          P.gC[i] = P.d_el * P.inv_h2;
          P.gMig[i] = P.t_plus * P.kappa * P.gF2;
        }
      } else if (k == K_CONTACT) {
        P.gP[i] = 2.0 * P.sig[a] * P.sig[b] / (P.sig[a] + P.sig[b]) * P.gF2;
      }
    }
  return P;
}

static const char* kPhaseName[6] = {"ELECTROLYTE", "GRAPHITE", "PLATED_LI", "LI_FOIL",
                                    "COLLECTOR_WORKING", "COLLECTOR_COUNTER"};

// scan a 0/1 int32 mask into a numbering (exclusive sum), -1 where mask is 0;
// optional inverse map; returns the count
static long long number_mask(const DBuf<int32_t>& mask, DBuf<int32_t>& num, DBuf<int32_t>* inv,
                             long long n, cudaStream_t s) {
  num.alloc(n);
  size_t tmp = 0;
  HC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, mask.p, num.p, (int64_t)n, s));
  DBuf<uint8_t> t(tmp);
  HC_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, mask.p, num.p, (int64_t)n, s));
  int32_t last_num = 0, last_mask = 0;
  HC_CUDA(cudaMemcpyAsync(&last_num, num.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaMemcpyAsync(&last_mask, mask.p + n - 1, 4, cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  long long count = (long long)last_num + last_mask;
  if (inv) inv->alloc(count);
  k_finalize_numbering<<<blocks_for(n), TPB, 0, s>>>(n, mask.p, num.p, inv ? inv->p : nullptr); HC_COUNT();
  HC_CHECK_LAUNCH();
  return count;
}

// ordered compaction of the face ids of one kind (reference face order)
static long long select_faces(const Operator& op, uint8_t kind, DBuf<long long>& out,
                              cudaStream_t s) {
  long long nx = op.P.nx, ny = op.P.ny, nz = op.P.nz;
  long long n_faces = (nz - 1) * ny * nx + nz * (ny - 1) * nx + nz * ny * (nx - 1);
  out.alloc(std::max<long long>(n_faces, 1));
  DBuf<long long> cnt(1);
  cub::CountingInputIterator<long long> it(0);
  FaceIsKind pred{op.P, op.labels.p, kind};
  size_t tmp = 0;
  HC_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, out.p, cnt.p, n_faces, pred, s));
  DBuf<uint8_t> t(tmp);
  HC_CUDA(cub::DeviceSelect::If(t.p, tmp, it, out.p, cnt.p, n_faces, pred, s));
  long long n = 0;
  HC_CUDA(cudaMemcpyAsync(&n, cnt.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
  HC_CUDA(cudaStreamSynchronize(s));
  return n;
}

Operator* create_operator(const uint8_t* labels_host, int nx, int ny, int nz, double voxel_um,
                          const hc_params& hp) {
  if (nx < 1 || ny < 1 || nz < 2) throw Error(HC_ERR_ARGUMENT, "grid must be at least 1x1x2");
  if (!(voxel_um > 0)) throw Error(HC_ERR_ARGUMENT, "voxel_size must be positive");
  long long nvox = (long long)nx * ny * nz;
  if (nvox >= (1LL << 31)) throw Error(HC_ERR_ARGUMENT, "grid exceeds 2^31 voxels");
  if (hp.n_ocp < 2 || hp.n_ocp > HC_MAX_OCP) throw Error(HC_ERR_ARGUMENT, "bad OCP table size");

  // phase presence checks on the host copy the caller handed us (dofmap.py:77-80, 87-89)
  long long cnt[6] = {0, 0, 0, 0, 0, 0};
  for (long long v = 0; v < nvox; ++v) {
    uint8_t a = labels_host[v];
    if (a >= 6) throw Error(HC_ERR_ARGUMENT, "label value out of range");
    cnt[a]++;
  }
  if (!cnt[GR]) throw Error(HC_ERR_MODEL, "grid contains no graphite electrode");
  if (!cnt[FOIL]) throw Error(HC_ERR_MODEL, "grid contains no lithium foil counter electrode");

  auto op = std::make_unique<Operator>();
  op->host_params = hp;
  op->voxel_um = voxel_um;
  op->P = make_dev_params(hp, nx, ny, nz, voxel_um);
  int dev = 0;
  HC_CUDA(cudaGetDevice(&dev));
  HC_CUDA(cudaDeviceGetAttribute(&op->n_sm, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t s = 0;
  const DevParams& P = op->P;

  HC_CUDA(cudaStreamCreateWithFlags(&op->stream, cudaStreamNonBlocking));
  if (const char* e = getenv("HC_KRYLOV_LOG")) op->krylov_log = atoi(e);
  if (const char* e = getenv("HC_DEV_KRYLOV")) op->dev_krylov = atoi(e) != 0;
  if (const char* e = getenv("HC_STENCIL")) op->stencil_kind = atoi(e);
  if (const char* e = getenv("HC_KRYLOV_BATCH")) op->krylov_batch = std::max(1, atoi(e));
  if (const char* e = getenv("HC_KRYLOV_WHILE")) op->krylov_while = atoi(e) != 0;
  if (const char* e = getenv("HC_NEWTON_DEV")) op->newton_dev = atoi(e) != 0;
  HC_CUDA(cudaEventCreateWithFlags(&op->ev_in, cudaEventDisableTiming));
  HC_CUDA(cudaEventCreateWithFlags(&op->ev_out, cudaEventDisableTiming));
  op->labels.alloc(nvox);
  HC_CUDA(cudaMemcpy(op->labels.p, labels_host, nvox, cudaMemcpyHostToDevice));


  // electrolyte path between electrode and counter electrode (dofmap.py:57-68,81-82)
  {
    DBuf<int32_t> par(nvox);
    DBuf<uint8_t> touch(((nvox + 3) / 4) * 4);
    DBuf<int> ok(1);
    HC_CUDA(cudaMemsetAsync(touch.p, 0, touch.n, s));
    HC_CUDA(cudaMemsetAsync(ok.p, 0, sizeof(int), s));
    k_uf_init<<<blocks_for(nvox), TPB, 0, s>>>(P, op->labels.p, par.p); HC_COUNT();
    k_uf_merge<<<blocks_for(nvox), TPB, 0, s>>>(P, op->labels.p, par.p); HC_COUNT();
    k_uf_touch<<<blocks_for(nvox), TPB, 0, s>>>(P, op->labels.p, par.p, touch.p); HC_COUNT();
    k_uf_both<<<blocks_for(nvox), TPB, 0, s>>>(nvox, touch.p, ok.p); HC_COUNT();
    HC_CHECK_LAUNCH();
    int okh = 0;
    HC_CUDA(cudaMemcpy(&okh, ok.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (!okh)
      throw Error(HC_ERR_MODEL,
                  "no electrolyte path connects the electrode to the counter electrode");
  }
  // outermost layer must hold counter collector to ground (dofmap.py:87-89)
  {
    bool any = false;
    const uint8_t* top = labels_host + (long long)(nz - 1) * nx * ny;
    for (long long i = 0; i < (long long)nx * ny; ++i) any |= top[i] == CC;
    if (!any) throw Error(HC_ERR_MODEL, "outermost z layer holds no counter collector to ground");
  }

  // DOF numbering (dofmap.py:84-97)
  DBuf<int32_t> cmask(nvox), pmask(nvox), plmask(nvox), plslot;
  k_masks<<<blocks_for(nvox), TPB, 0, s>>>(P, op->labels.p, cmask.p, pmask.p, plmask.p); HC_COUNT();
  HC_CHECK_LAUNCH();
  op->info.n_c = number_mask(cmask, op->cdof, &op->c_vox, nvox, s);
  op->info.n_p = number_mask(pmask, op->pdof, &op->p_vox, nvox, s);
  op->info.n_plated = number_mask(plmask, plslot, &op->plated_vox, nvox, s);
  op->info.n_dirichlet = nvox - op->info.n_p;

  // forbidden adjacency / kinetics on grounded faces (operator.py:145-168)
  long long n_faces = (long long)(nz - 1) * ny * nx + (long long)nz * (ny - 1) * nx +
                      (long long)nz * ny * (nx - 1);
  {
    DBuf<int> err(1);
    DBuf<unsigned long long> bad(1);
    HC_CUDA(cudaMemset(err.p, 0, sizeof(int)));
    HC_CUDA(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
    if (n_faces)
      k_face_check<<<blocks_for(n_faces), TPB, 0, s>>>(P, op->labels.p, n_faces, err.p, bad.p); HC_COUNT();
    HC_CHECK_LAUNCH();
    int e = 0;
    unsigned long long fb = 0;
    HC_CUDA(cudaMemcpy(&e, err.p, sizeof(int), cudaMemcpyDeviceToHost));
    HC_CUDA(cudaMemcpy(&fb, bad.p, sizeof(fb), cudaMemcpyDeviceToHost));
    if (e & 1) {
      // recompute the offending pair on the host for the message
      long long f = (long long)fb, lo, hi;
      long long fz = (long long)(nz - 1) * ny * nx, fy = (long long)nz * (ny - 1) * nx;
      if (f < fz) { lo = f; hi = f + (long long)ny * nx; }
      else if (f < fz + fy) {
        long long g = f - fz, x = g % nx, t = g / nx, y = t % (ny - 1), z = t / (ny - 1);
        lo = (z * ny + y) * nx + x; hi = lo + nx;
      } else {
        long long g = f - fz - fy, x = g % (nx - 1), t = g / (nx - 1), y = t % ny, z = t / ny;
        lo = (z * ny + y) * nx + x; hi = lo + 1;
      }
      throw Error(HC_ERR_MODEL, std::string(kPhaseName[labels_host[lo]]) + " and " +
                                    kPhaseName[labels_host[hi]] +
                                    " voxels share a face; this adjacency is geometrically "
                                    "forbidden");
    }
    if (e & 2)
      throw Error(HC_ERR_MODEL, "interface kinetics on a grounded face are not supported");
  }

  // compacted interface face lists, unified as [bv | ce | strip] (operator.py:210-219)
  DBuf<long long> fbv, fce, fst;
  long long nbv = select_faces(*op, K_BV, fbv, s);
  long long nce = select_faces(*op, K_CE, fce, s);
  long long nst = select_faces(*op, K_STRIP, fst, s);
  op->info.n_bv = nbv;
  op->info.n_ce = nce;
  op->info.n_strip = nst;
  op->n_if = nbv + nce + nst;
  op->if_solid.alloc(op->n_if);
  op->if_el.alloc(op->n_if);
  op->if_slot.alloc(op->n_if);
  op->if_kind.alloc(op->n_if);
  long long off = 0;
  const DBuf<long long>* lists[3] = {&fbv, &fce, &fst};
  long long ns[3] = {nbv, nce, nst};
  for (int k = 0; k < 3; ++k) {
    if (ns[k])
      k_orient<<<blocks_for(ns[k]), TPB, 0, s>>>(P, op->labels.p, lists[k]->p, ns[k], (int8_t)k,
                                                 plslot.p, op->if_solid.p + off,
                                                 op->if_el.p + off, op->if_slot.p + off,
                                                 op->if_kind.p + off); HC_COUNT();
    off += ns[k];
  }
  HC_CHECK_LAUNCH();
  // voxel -> (direction -> interface face) map for deterministic per-voxel gathers
  {
    DBuf<int32_t> mark(nvox);
    HC_CUDA(cudaMemsetAsync(mark.p, 0, nvox * sizeof(int32_t), s));
    if (op->n_if)
      k_if_mark<<<blocks_for(op->n_if), TPB, 0, s>>>(op->n_if, op->if_solid.p, op->if_el.p,
                                                      mark.p); HC_COUNT();
    HC_CHECK_LAUNCH();
    long long n_ifv = number_mask(mark, op->if_rank, nullptr, nvox, s);
    op->if_dir.alloc(std::max<long long>(6 * n_ifv, 1));
    HC_CUDA(cudaMemsetAsync(op->if_dir.p, 0xff, op->if_dir.n * sizeof(int32_t), s));
    if (op->n_if)
      k_if_dirs<<<blocks_for(op->n_if), TPB, 0, s>>>(P, op->n_if, op->if_solid.p, op->if_el.p,
                                                      op->if_rank.p, op->if_dir.p); HC_COUNT();
    HC_CHECK_LAUNCH();
  }
  // 32-bit labels for the staged stencils: phase | (interface rank + 1) << 3
  {
    std::vector<int32_t> rank(nvox), l4(nvox);
    HC_CUDA(cudaMemcpy(rank.data(), op->if_rank.p, nvox * 4, cudaMemcpyDeviceToHost));
    for (long long v = 0; v < nvox; ++v) l4[v] = (int32_t)labels_host[v] | ((rank[v] + 1) << 3);
    op->lab4.alloc(nvox);
    HC_CUDA(cudaMemcpy(op->lab4.p, l4.data(), nvox * 4, cudaMemcpyHostToDevice));
    if (tma_grid_ok(P)) {
      // TMA face word (hc_tma.cuh): (phase + 1) | interface mask << 3 | same-phase
      // conduction mask << 9 | contact flag | grounded-row flag | tile-plane-local first
      // slot << 17 — phase + 1 so that the TMA zero fill reads as "outside"; the slots of a
      // voxel's interface faces are consecutive in direction order
      std::vector<int32_t> dirs(op->if_dir.n);
      HC_CUDA(cudaMemcpy(dirs.data(), op->if_dir.p, dirs.size() * 4, cudaMemcpyDeviceToHost));
      // per interface face: its slot on the solid side and on the electrolyte side
      std::vector<int2> fslot(std::max<long long>(op->n_if, 1), make_int2(0, 0));
      // slots numbered tile-plane by tile-plane (32 x 8 tile, plane z), so the slots a
      // TMA stencil CTA needs for one plane are one contiguous block (bulk-copied by its
      // producer warp); tp_off[tile-plane] = first slot of that block
      const int tbx0 = (nx + VX - 1) / VX, tby0 = (ny + VY - 1) / VY;
      std::vector<int32_t> tp_off((size_t)tbx0 * tby0 * nz + 1, 0);
      long long slot = 0;
      bool fits = true;
      for (int z = 0; z < nz; ++z)
        for (int ty = 0; ty < tby0; ++ty)
          for (int tx = 0; tx < tbx0; ++tx) {
            const long long tp0 = slot;
            tp_off[((size_t)z * tby0 + ty) * tbx0 + tx] = (int32_t)slot;
            for (int y = ty * VY; y < std::min(ny, ty * VY + VY); ++y)
              for (int x = tx * VX; x < std::min(nx, tx * VX + VX); ++x) {
                const long long v = ((long long)z * ny + y) * nx + x;
                const uint8_t a = labels_host[v];
                int mask = 0, smask = 0, contact = 0;
                const long long nb[6] = {x > 0 ? v - 1 : -1, x + 1 < nx ? v + 1 : -1,
                                         y > 0 ? v - nx : -1, y + 1 < ny ? v + nx : -1,
                                         z > 0 ? v - (long long)nx * ny : -1,
                                         z + 1 < nz ? v + (long long)nx * ny : -1};
                for (int d = 0; d < 6; ++d) {
                  if (nb[d] < 0) continue;
                  const uint8_t k = kind_of(a, labels_host[nb[d]]);
                  if (k == K_CONT) smask |= 1 << d;
                  if (k == K_CONTACT) contact = 1;
                }
                if (rank[v] >= 0)
                  for (int d = 0; d < 6; ++d) {
                    const int32_t f = dirs[6LL * rank[v] + d];
                    if (f < 0) continue;
                    mask |= 1 << d;
                    if (a == EL) fslot[f].y = (int)(slot + __builtin_popcount(mask) - 1);
                    else fslot[f].x = (int)(slot + __builtin_popcount(mask) - 1);
                  }
                const long long loc = slot - tp0;
                if (loc >= (1LL << 15) || slot + 6 >= (1LL << 31)) fits = false;
                const int grounded = (z == nz - 1 && a == CC) ? 1 : 0;
                l4[v] = (int32_t)((uint32_t)(a + 1) | (uint32_t)mask << 3 | (uint32_t)smask << 9 |
                                  (uint32_t)contact << 15 | (uint32_t)grounded << 16 |
                                  (uint32_t)(loc & 0x7fff) << 17);
                slot += __builtin_popcount(mask);
              }
          }
      tp_off.back() = (int32_t)slot;
      if (fits) {
        op->labt.alloc(nvox);
        HC_CUDA(cudaMemcpy(op->labt.p, l4.data(), nvox * 4, cudaMemcpyHostToDevice));
        op->if_cslot.alloc(std::max<long long>(4 * slot, 2));
        HC_CUDA(cudaMemset(op->if_cslot.p, 0, op->if_cslot.n * sizeof(double)));
        op->tp_off.alloc(tp_off.size());
        HC_CUDA(cudaMemcpy(op->tp_off.p, tp_off.data(), tp_off.size() * 4, cudaMemcpyHostToDevice));
        op->if_islot.alloc(std::max<long long>(slot, 1));
        HC_CUDA(cudaMemset(op->if_islot.p, 0, op->if_islot.n * sizeof(double)));
        op->if_fslot.alloc(fslot.size());
        HC_CUDA(cudaMemcpy(op->if_fslot.p, fslot.data(), fslot.size() * sizeof(int2), cudaMemcpyHostToDevice));
        const int tbx = (nx + VX - 1) / VX, tby = (ny + VY - 1) / VY;
        std::vector<int2> ez(tbx * tby, make_int2(nz, -1));
        for (long long v = 0; v < nvox; ++v)
          if (labels_host[v] == EL) {
            const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((long long)nx * ny));
            int2& t = ez[(y / VY) * tbx + x / VX];
            t.x = std::min(t.x, z);
            t.y = std::max(t.y, z);
          }
        {
          int zlo = nz, zhi = -1;
          for (int z = 0; z < nz; ++z) {
            bool any = false;
            for (long long v = (long long)z * nx * ny; v < (long long)(z + 1) * nx * ny && !any; ++v)
              any = labels_host[v] == EL || labels_host[v] == GR;
            if (any) {
              zlo = std::min(zlo, z);
              zhi = std::max(zhi, z);
            }
          }
          op->cz = zhi >= zlo ? make_int2(zlo, zhi + 1) : make_int2(0, 0);
        }
        op->elz.alloc(ez.size());
        HC_CUDA(cudaMemcpy(op->elz.p, ez.data(), ez.size() * sizeof(int2), cudaMemcpyHostToDevice));
        op->tma = new TmaCache();
      }
    }
  }
  // electrolyte-electrolyte faces (operator.py:187-191), kept for export
  {
    DBuf<long long> fel;
    long long n_elel = select_faces(*op, 7, fel, s);
    op->info.n_elel = n_elel;
    op->elel_lo.alloc(n_elel);
    op->elel_hi.alloc(n_elel);
    if (n_elel)
      k_elel_pairs<<<blocks_for(n_elel), TPB, 0, s>>>(P, fel.p, n_elel, op->elel_lo.p,
                                                      op->elel_hi.p); HC_COUNT();
    HC_CHECK_LAUNCH();
  }
  // drive faces: working-collector voxels in the z = 0 layer (operator.py:229-235)
  {
    long long nd = 0;
    for (long long i = 0; i < (long long)nx * ny; ++i) nd += labels_host[i] == CW;
    op->info.n_drive_faces = nd;
  }
  op->info.nx = nx;
  op->info.ny = ny;
  op->info.nz = nz;
  op->info.n_vox = nvox;
  op->info.h = P.h;
  op->info.face_area = P.h * P.h;
  op->info.voxel_volume = P.h * P.h * P.h;
  op->info.n_const = P.n_const;
  op->info.scale = P.sc;

  // work space
  op->xg.alloc(nvox);
  op->xg2.alloc(nvox);
  op->vg.alloc(nvox);
  op->outg.alloc(nvox);
  op->cprev.alloc(nvox);
  op->inv_c.alloc(nvox);
  op->if_coef.alloc(std::max<long long>(3 * op->n_if, 1));
  op->if_cur.alloc(std::max<long long>(op->n_if, 1));
  op->if_vcoef.alloc(3 * op->if_dir.n);
  HC_CUDA(cudaMemset(op->if_vcoef.p, 0, op->if_vcoef.n * sizeof(double)));
  op->npl.alloc(std::max<long long>(op->info.n_plated, 1));
  op->red.alloc(4096);
  HC_CUDA(cudaDeviceSynchronize());
  return op.release();
}

void set_params(Operator& op, const hc_params& hp) {
  HC_CUDA(cudaDeviceSynchronize());
  op.host_params = hp;
  op.P = make_dev_params(hp, op.P.nx, op.P.ny, op.P.nz, op.voxel_um);
  op.info.n_const = op.P.n_const;
  op.info.scale = op.P.sc;
}

}  // namespace hc
