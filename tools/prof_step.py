"""Profiling driver: set up a config, warm one step, then run ONE profiled step
between cudaProfilerStart/Stop (use with ncu --profile-from-start off)."""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import _dev, _native
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
name = sys.argv[1] if len(sys.argv) > 1 else 'large'
rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
op = P.SystemOperator(P.build_dofmap(grid), params)
h = grid.voxel_size * 1e-6
mu = -rs.c_rate * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) * h**3 / 3600 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
import os
cfg = P.SolverConfig(dt_max=rs.dt, dt_init=min(0.05, rs.dt), linear_safety=float(os.environ.get('LS', '0.1')))
st = P.prepare_initial_state(op, params, mu, cfg)
x = _dev.to_dev(st.x).clone(); npl = _dev.to_dev(st.n_pl).clone()
c = cfg.to_c(); s = _native.HcNewtonStats()
L = _native.lib()
def step():
    _native.check(L.hc_step(op.native.handle, _dev.ptr(x), _dev.ptr(npl), 0.0, rs.dt, mu, ctypes.byref(c), ctypes.byref(s), None))
step(); torch.cuda.synchronize()
t = time.time(); step(); torch.cuda.synchronize(); print('warm step %.3f s newton %d krylov %d' % (time.time() - t, s.n_iter, s.krylov_iters), flush=True)
torch.cuda.profiler.start()
step(); torch.cuda.synchronize()
torch.cuda.profiler.stop()
print('profiled step: newton %d krylov %d' % (s.n_iter, s.krylov_iters))
