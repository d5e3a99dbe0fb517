"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  It is the checker, never the thing measured or
shipped: the product package (paper_2505_01968_b200) does not import it.

Contents
  rapp_oracle.c / liboracle.so  plain-C restatement of the reference table path
  _ref/_grid_cy*.so             the reference's own compiled Cython kernel
  scaler_oracle.py              pure-Python restatement of Autoscaler.scale and
                                the per-tick loop (small cases)
"""

from .binding import (load_oracle, load_reference_kernel, or_interp3, or_interp3_many,
                      or_locate, or_most_efficient_config)

__all__ = ["load_oracle", "load_reference_kernel", "or_interp3", "or_interp3_many",
           "or_locate", "or_most_efficient_config"]
