"""B200-native full-order implicit step of the microstructure-resolved half-cell
model (arXiv 1704.04139), drop-in for the reference package ``halfcell``'s
``fvm`` entry points.  Compute runs in ``libhalfcell_b200.so`` (CUDA, sm_100a);
there is no CPU fallback."""

from .errors import (ConfigError, DomainError, GeometryError, HalfcellError, ModelError,
                     NativeError, NonConvergence, NumericsError, ReductionError,
                     SimulationError)
from .params import DEFAULT_OCP_TABLE, FARADAY, GAS_CONSTANT, MaterialParams, PhysConstants
from .phases import N_PHASES, Phase, PhaseGrid

__version__ = "0.1.0"

_LAZY = {
    "Dofmap": "dofmap", "build_dofmap": "dofmap",
    "SystemOperator": "system_operator", "BoundaryDrive": "system_operator",
    "SolverConfig": "newton", "NewtonResult": "newton", "newton_solve": "newton",
    "solve_initial_potential": "newton",
    "CellState": "state", "initial_fields": "state",
    "StepInfo": "timestepping", "Trajectory": "timestepping", "step": "timestepping",
    "prepare_initial_state": "timestepping", "run_transient": "timestepping",
    "qoi_vectors": "qoi", "qoi_cell_voltage": "qoi", "qoi_mean_solid_conc": "qoi",
    "pod_gram": "pod", "pod_basis": "pod",
    "make_batch": "batch", "step_batch": "batch", "BatchCell": "batch",
    "SubOperatorView": "suboperator", "RestrictedSubOperator": "suboperator",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib
        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
