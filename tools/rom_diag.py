"""Scratch: snapshot health of the ROM bench workload (medium cell) under the current env."""
import sys, os, ctypes
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import mor, _native, _dev
from paper_1704_04139_b200.microgen import generate_cell
import bench
rs, spec = bench.cell_for("medium", 0)
grid = generate_cell(spec)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
op = P.SystemOperator(P.build_dofmap(grid), params)
mu = bench.drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
dt = rs.dt
cfg = P.SolverConfig(dt_init=min(0.05, dt), dt_max=dt, linear_safety=bench.LINEAR_SAFETY)
st = P.prepare_initial_state(op, params, mu, cfg)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
c = P.SolverConfig(dt_init=dt, dt_max=dt, linear_safety=bench.LINEAR_SAFETY).to_c()
x = _dev.to_dev(st.x).clone(); npl = _dev.to_dev(st.n_pl if st.n_pl.size else np.zeros(1)).clone()
s = _native.HcNewtonStats()
bad = 0
for k in range(n):
    _native.check(_native.lib().hc_step(op.native.handle, _dev.ptr(x), _dev.ptr(npl), 0.0, dt, float(mu), ctypes.byref(c), ctypes.byref(s), _dev.stream()))
    fin = bool(torch.isfinite(x).all())
    if k % 50 == 0 or not fin or s.dt_used != dt or s.retries:
        print(k, "dt_used", s.dt_used, "newton", s.n_iter, "krylov", s.krylov_iters, "retries", s.retries, "finite", fin, "norm", float(x.norm()), flush=True)
    if not fin:
        break
print("npl finite", bool(torch.isfinite(npl).all()), "x norm", float(x.norm()))
