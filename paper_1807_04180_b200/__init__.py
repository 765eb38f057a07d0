"""B200-native (sm_100a) DDM hot path for the high-frequency Helmholtz equation
(arXiv 1807.04180): batched supernodal PML solves, fused source transfer and
device-resident FGMRES behind the reference's DdmEngine / fgmres surface.

The compute lives in ``libhddm.so`` (CUDA, built in-tree by
``__graft_entry__.build()``); this package is the host-side mirror of the
reference interface (``engine.DdmEngine``) and the shared input generator
(``problems``).
"""
from .problems import Problem, config, small, random_layers  # noqa: F401


def __getattr__(name):
    # engine symbols are resolved lazily so that importing the package (for the
    # problem generator) does not require the CUDA library
    if name in ("DdmEngine", "DdmStats", "FgmresOptions", "FgmresResult", "ConfigError",
                "SolveError", "HddmError", "load_library", "nd_order"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
