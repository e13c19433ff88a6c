"""Python step() API rate vs the C-ABI host-buffer step on a BASELINE config (GPU box).

    python tools/step_api_rate.py [config] [steps]
"""
import ctypes, sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import _native
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
name = sys.argv[1] if len(sys.argv) > 1 else 'large'
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
op = P.SystemOperator(P.build_dofmap(grid), params)
h = grid.voxel_size * 1e-6
mu = -rs.c_rate * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) * h**3 / 3600 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
kw = dict(newton_rtol=1e-8, linear_rtol=1e-10) if name == 'large' else {}
cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, **kw)
st0 = P.prepare_initial_state(op, params, mu, cfg)
st, *_ = P.step(op, st0, rs.dt, mu, cfg)
t = time.perf_counter()
for _ in range(n):
    st, *_ = P.step(op, st, rs.dt, mu, cfg)
api = n / (time.perf_counter() - t)
sd = st0.to_device()
sd, *_ = P.step(op, sd, rs.dt, mu, cfg)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(n):
    sd, *_ = P.step(op, sd, rs.dt, mu, cfg)
torch.cuda.synchronize(); dev = n / (time.perf_counter() - t)
xh = torch.from_numpy(st0.x.copy()).pin_memory(); nh = torch.from_numpy(st0.n_pl.copy()).pin_memory()
c = cfg.to_c(); s = _native.HcNewtonStats(); L = _native.lib()
L.hc_step_host(op.native.handle, xh.data_ptr(), nh.data_ptr(), 0.0, rs.dt, mu, ctypes.byref(c), ctypes.byref(s))
t = time.perf_counter()
for _ in range(n):
    _native.check(L.hc_step_host(op.native.handle, xh.data_ptr(), nh.data_ptr(), 0.0, rs.dt, mu, ctypes.byref(c), ctypes.byref(s)))
host = n / (time.perf_counter() - t)
print(f"{name}: step() numpy state {api:.2f} steps/s, step() device state {dev:.2f}, hc_step_host {host:.2f}; "
      f"ratio numpy/host {api / host:.3f}")
