"""B200-native component-wise solver-free ADMM for LinDistFlow OPF (arXiv 2501.08293).

Drop-in for the reference's `dopf::solve` hot path: host C++ front-end
(libdopf_host.so) + hand-written sm_100a fp64 kernels (libdopf_cuda.so).
"""
from . import dopf  # noqa: F401
from .dopf import (  # noqa: F401
    Settings, SolveResult, solve, parse_feeder, parse_feeder_file, validate_feeder,
    assemble_centralized, decompose, synthetic_feeder, tiled_feeder, scale_loads,
    CudaSolver, ParseError, SingularSubsystemError, InfeasibleSubsystemError,
)
