"""B200-native RaPP prediction + hybrid-autoscaler decision path.

Drop-in for the hot path of the reference package `hybridscale` (HAS-GPU,
arxiv 2505.01968): the table kernel module (`kernels`), the performance model
(`perf.PerfTable`, `perf.PerfTableSet`), and the scaler decision procedure
(`autoscaler`, `tick`).  All predictions and searches run on the GPU through
librapp_b200.so (include/rapp_b200.h); there is no CPU fallback.
"""

from . import errors
from .perf import (PerfModel, PerfTable, PerfTableSet, load_table, save_table,
                   validate_table_file)

KERNEL_BACKEND = "b200"

__version__ = "0.1.0"

__all__ = ["KERNEL_BACKEND", "PerfModel", "PerfTable", "PerfTableSet", "errors", "load_table",
           "save_table", "validate_table_file"]
