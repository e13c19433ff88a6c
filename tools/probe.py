"""Scratch probe: build a BASELINE cell, initial potential, a few steps, print timings."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1704_04139_b200 as P
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
import torch

name = sys.argv[1] if len(sys.argv) > 1 else 'tiny'
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rs = CONFIGS[name]
t = time.time(); grid = generate_cell(rs.cell); print('gen', time.time() - t, flush=True)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
t = time.time(); dof = P.build_dofmap(grid); op = P.SystemOperator(dof, params); print('setup', time.time() - t, dof.describe(), flush=True)
flat = grid.labels.ravel()
vol_gr = (flat == 1).sum() * (grid.voxel_size * 1e-6) ** 3
area = grid.labels.shape[1] * grid.labels.shape[2] * (grid.voxel_size * 1e-6) ** 2
mu = -rs.c_rate * params.c_gr_max * params.constants.F * vol_gr / 3600 / area
print('mu', mu)
cfg = P.SolverConfig(dt_max=rs.dt, dt_init=min(0.05, rs.dt))
t = time.time(); st = P.prepare_initial_state(op, params, mu, cfg); torch.cuda.synchronize(); print('init potential', time.time() - t, flush=True)
v_cp, v_ac = P.qoi_vectors(dof)
for k in range(nsteps):
    t = time.time()
    st, dt, dtn, info = P.step(op, st, rs.dt, mu, cfg)
    print(f'step {k} {time.time()-t:.3f}s V={v_cp@st.x:.6f} cbar={v_ac@st.x:.3f} npl={st.n_pl.sum():.4e} {info}', flush=True)
