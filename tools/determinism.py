"""Scratch: is a run of full-order steps bitwise reproducible (same process, fresh operators)?"""
import sys, os, hashlib
sys.path.insert(0, '.')
import numpy as np
import paper_1704_04139_b200 as P
from paper_1704_04139_b200.microgen import generate_cell
import bench
rs, spec = bench.cell_for("medium", 0)
grid = generate_cell(spec)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
mu = bench.drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
for rep in range(2):
    op = P.SystemOperator(P.build_dofmap(grid), params)
    cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=0.3)
    st = P.prepare_initial_state(op, params, mu, cfg)
    h0 = hashlib.sha1(st.x.tobytes()).hexdigest()[:12]
    dt = rs.dt
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
        st, _, _, info = P.step(op, st, dt, mu, cfg)
    print(rep, "init", h0, "after", hashlib.sha1(st.x.tobytes()).hexdigest()[:12], flush=True)
