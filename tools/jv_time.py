"""CUDA-event times of the residual / J v kernels of a config (bench.py's kernel_roofline leg only).
Usage: jv_time.py [config] [iters]"""
import ctypes, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1704_04139_b200 as P
from paper_1704_04139_b200 import _dev, _native
from paper_1704_04139_b200.configs import CONFIGS
from paper_1704_04139_b200.microgen import generate_cell
from paper_1704_04139_b200.state import initial_fields
name = sys.argv[1] if len(sys.argv) > 1 else 'large'
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rs = CONFIGS[name]
grid = generate_cell(rs.cell)
params = P.MaterialParams(soc_init=rs.soc_init, i00_plel=rs.i00_plel_exchange / np.sqrt(1000.0))
dof = P.build_dofmap(grid)
op = P.SystemOperator(dof, params)
st = initial_fields(dof, params)
x = _dev.to_dev(st.x); npl = _dev.to_dev(st.n_pl if st.n_pl.size else np.zeros(1))
beta = rs.dt * op.face_area / params.constants.F
L = _native.lib()
ms = (ctypes.c_double * 5)()
_native.check(L.hc_time_kernels(op.native.handle, _dev.ptr(x), _dev.ptr(npl), beta, 1.0 / rs.dt, iters, 256 << 20, ms, _dev.stream()))
info = op.native.info
nvox = int(info.n_vox); n_el = int(np.count_nonzero(grid.labels == 0)); n_c = int(np.count_nonzero(np.isin(grid.labels, (0, 1))))
n_if = int(info.n_bv + info.n_ce + info.n_strip)
jb = nvox * 33 + n_el * 8 + n_if * 24; rb = nvox * 33 + n_c * 8
print(f"{name}: residual {ms[0]*1e3:.1f} + {ms[1]*1e3:.1f} us ({rb/(ms[0]+ms[1])/1e6:.0f} GB/s)  jv {ms[2]*1e3:.1f} us ({jb/ms[2]/1e6:.0f} GB/s, frac {jb/ms[2]/1e6/6543.7:.3f})  copy {ms[4]*1e3:.1f} us  n_if {n_if}")
