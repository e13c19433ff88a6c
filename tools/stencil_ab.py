"""Scratch A/B: J v / residual / sweep timings and results per stencil kind (HC_STENCIL)
on one config.  Usage: python tools/stencil_ab.py large [kinds...]"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import _dev, _native
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell

name = sys.argv[1] if len(sys.argv) > 1 else "large"
kinds = [int(k) for k in sys.argv[2:]] or [2, 3]
rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
dof = P.build_dofmap(grid)
rng = np.random.default_rng(0)
res = {}
for k in kinds:
    os.environ["HC_STENCIL"] = str(k)
    op = P.SystemOperator(dof, params)
    from paper_1704_04139_b200.state import initial_fields
    st = initial_fields(dof, params)
    x = st.x.copy()
    nc = dof.n_c
    x[:nc] *= 1.0 + 0.05 * rng.standard_normal(nc) if k == kinds[0] else 1.0
    if k == kinds[0]:
        x0 = x.copy()
        v0 = rng.standard_normal(dof.n_total)
    x = x0
    npl = st.n_pl if st.n_pl.size else np.zeros(1)
    beta = rs.dt * op.face_area / params.constants.F
    jv = op.jvp(x, npl, v0, beta=beta, inv_dt=1.0 / rs.dt)
    r = op.apply(x, npl, -1.0, beta=beta)
    ms = (ctypes.c_double * 5)()
    xd, nd = _dev.to_dev(x), _dev.to_dev(npl)
    _native.check(_native.lib().hc_time_kernels(op.native.handle, _dev.ptr(xd), _dev.ptr(nd), beta,
                                                1.0 / rs.dt, 20, int(os.environ.get("FLUSH_MB", "256")) << 20, ms, _dev.stream()))
    nvox = grid.labels.size
    print(f"kind {k}: residual {ms[0]*1e3:.1f}+{ms[1]*1e3:.1f} us, jv {ms[2]*1e3:.1f}+{ms[3]*1e3:.1f} us, "
          f"copy {ms[4]*1e3:.1f} us ({nvox*32/ms[4]/1e6:.0f} GB/s)", flush=True)
    res[k] = (jv, r)
    del op
if len(kinds) > 1:
    a, b = res[kinds[0]], res[kinds[1]]
    sc = np.maximum(np.abs(a[0]), 1e-300)
    print("jv max rel diff", float(np.max(np.abs(a[0] - b[0]) / np.maximum(np.abs(a[0]).max(), 1e-300))),
          "max abs", float(np.max(np.abs(a[0] - b[0]))), "bitwise equal", bool(np.array_equal(a[0], b[0])))
    print("res bitwise equal", bool(np.array_equal(a[1], b[1])))
