"""Scratch: Krylov iteration counts of the device solver under AMG knob settings."""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import _dev, _native
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
import torch
name = sys.argv[1]
settings = [s.split(',') for s in sys.argv[2:]] or [['2', '0.6', '1.0']]
import dataclasses
if name == 'thick32':
    rs = dataclasses.replace(CONFIGS['large'], cell=dataclasses.replace(CONFIGS['large'].cell, nx=32, ny=32, nz=256, n_anode=200, n_separator=32))
elif name.startswith('large') and name != 'large':
    w = int(name[5:])
    rs = dataclasses.replace(CONFIGS['large'], cell=dataclasses.replace(CONFIGS['large'].cell, nx=w, ny=w))
else:
    rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
dof = P.build_dofmap(grid)
h = grid.voxel_size * 1e-6
mu = -rs.c_rate * params.c_gr_max * params.constants.F * np.count_nonzero(grid.labels == 1) * h**3 / 3600 / (grid.labels.shape[1] * grid.labels.shape[2] * h * h)
from paper_1704_04139_b200.state import initial_fields
st0 = initial_fields(dof, params)
for nu, om, al in settings:
    os.environ['HC_AMG_NU'], os.environ['HC_AMG_OMEGA'], os.environ['HC_AMG_ALPHA'] = nu, om, al
    op = P.SystemOperator(dof, params)
    cfg = P.SolverConfig(dt_max=rs.dt, dt_init=min(0.05, rs.dt))
    c = cfg.to_c(); stt = _native.HcNewtonStats()
    x = _dev.to_dev(st0.x); npl = _dev.to_dev(st0.n_pl); out = _dev.empty(dof.n_total)
    t = time.time()
    _native.check(_native.lib().hc_solve_initial_potential(op.native.handle, _dev.ptr(x), _dev.ptr(npl), mu, ctypes.byref(c), _dev.ptr(out), ctypes.byref(stt), None))
    t_init = time.time() - t
    ki = stt.krylov_iters; ni = stt.n_iter
    xs = out.clone(); ns = npl.clone()
    t = time.time(); ks = []
    for k in range(2):
        _native.check(_native.lib().hc_step(op.native.handle, _dev.ptr(xs), _dev.ptr(ns), 0.0, rs.dt, mu, ctypes.byref(c), ctypes.byref(stt), None))
        ks.append((stt.n_iter, stt.krylov_iters))
    torch.cuda.synchronize()
    print(f'nu={nu} omega={om} alpha={al}: init {ni} newton / {ki} krylov in {t_init:.2f}s; steps {ks} in {time.time()-t:.2f}s', flush=True)
    del op
