"""B200-native hot path of the arXiv 1704.01144 LTS finite-volume solver.

The product is ``libtafv_gpu.so`` (CUDA sm_100a kernels + C++ runtime behind
the C ABI of ``include/tafv_gpu.h``); this package is the thin Python host
mirror used by the tests and the benchmark.
"""
from .api import (CudaError, Diverged, InvalidArgument, LogicError, Solver,  # noqa: F401
                  SolverOptions, TafvError)

__all__ = ["Solver", "SolverOptions", "InvalidArgument", "LogicError", "Diverged", "CudaError",
           "TafvError"]
