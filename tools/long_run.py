"""Robustness run: a BASELINE config for its full step count on the GPU (fixed dt),
printing the QoI curve endpoints, Newton/Krylov totals and the wall time."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "large"
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].n_steps
rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
op = P.SystemOperator(P.build_dofmap(grid), params)
mu = bench.drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
cfg = P.SolverConfig(dt_init=min(0.05, rs.dt), dt_max=rs.dt, linear_safety=bench.LINEAR_SAFETY)
st = P.prepare_initial_state(op, params, mu, cfg)
v_cp, v_ac = P.qoi_vectors(op.dof)
t0 = time.time()
newton = krylov = 0
vs = []
while st.t < n_steps * rs.dt - 1e-9:
    st, dt_used, _, info = P.step(op, st, min(rs.dt, n_steps * rs.dt - st.t), mu, cfg)
    newton += info.n_iter
    krylov += info.krylov_iters
    vs.append(v_cp @ st.x)
torch.cuda.synchronize()
el = time.time() - t0
print(f"{name}: t_end={st.t:.3f}s steps={len(vs)} wall={el:.2f}s ({len(vs)/el:.2f} steps/s incl. host I/O) "
      f"newton={newton} krylov={krylov} V: {vs[0]:.6f} -> {vs[-1]:.6f}  mean c_s: {v_ac @ st.x:.3f}  "
      f"plated: {st.n_pl.sum():.4e}")
