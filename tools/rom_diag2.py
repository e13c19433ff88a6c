"""Scratch: spectra and EI conditioning of the ROM bench build under the current env."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import mor
from paper_1704_04139_b200.microgen import generate_cell
import bench
rs, spec = bench.cell_for("medium", 0)
grid = generate_cell(spec)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
op = P.SystemOperator(P.build_dofmap(grid), params)
mu = bench.drive_mu(grid.labels, grid.voxel_size, rs.c_rate, params)
dt = rs.dt
st = P.prepare_initial_state(op, params, mu, P.SolverConfig(dt_init=min(0.05, dt), dt_max=dt, linear_safety=bench.LINEAR_SAFETY))
import os
snaps = mor.collect_snapshots(op, st.x, st.n_pl, mu, dt, 400, P.SolverConfig(dt_init=dt, dt_max=dt, linear_safety=float(os.environ.get("SNAP_SAFETY", "0"))))
nc = op.dof.n_c
idx = [0, 20, 40, 59, 100, 150, 200, 250, 299, 350]
for name, S, k in (("c", snaps.X[:nc], 60), ("phi", snaps.X[nc:], 60), ("N", snaps.N, 300)):
    V, sig = mor.pod_rank(S, k)
    s = sig.cpu().numpy()
    print(name, "kept", V.shape[1], " ".join(f"{i}:{s[i]/s[0]:.1e}" for i in idx if i < s.size), flush=True)
    if name == "N":
        W = V
        pi = mor.deim(W)
        Wp = W[torch.as_tensor(pi, device="cuda")]
        sv = torch.linalg.svdvals(Wp).cpu().numpy()
        print("cond W_pi", sv[0] / sv[-1], "smallest", sv[-1])
        for mm in (100, 150, 200, 250):
            piw = mor.deim(W[:, :mm].contiguous())
            sv = torch.linalg.svdvals(W[:, :mm][torch.as_tensor(piw, device='cuda')]).cpu().numpy()
            print(" m", mm, "cond", sv[0] / sv[-1])
try:
    rom = mor.build_rom(op, snaps, 60, 60, 300)
    tr = mor.solve_rom(op, rom, rom.project(st.x), st.n_pl, mu, dt, 5)
    print("rom ok", tr.voltage[:3])
except Exception as e:
    print("rom failed:", e)
