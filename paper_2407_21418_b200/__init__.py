"""B200-native FTuner hot path: dynamic-shape Dense / BatchMatmul executed as a
patchwork of variously-sized uKernels on sm_100a (tcgen05 + TMA + TMEM).

Subpackages / modules:
  mktune/    drop-in facade of the reference package's tuner API (same module,
             function and class names as mktune 0.1.0), backed by the C++
             planner in libftb.so
  execute    ProgramPlan -> tile-schedule table -> one persistent kernel launch
  _lib       ctypes binding of libftb.so (include/ftb.h)
"""

__version__ = "0.1.0"
