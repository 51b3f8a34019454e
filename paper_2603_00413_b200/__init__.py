"""B200-native (sm_100a) differentiable recursive mesh ray tracer of DiffTrans
(arXiv 2603.00413, refine stage).  See DESIGN.md and include/difftrans.h.

Modules:
  scenes   seeded synthetic inputs (shared with the tests' oracle; no method arithmetic)
  tracer   torch front-end of the C ABI (Tracer, DeviceScene, DiffTraceFunction)
  dist     view/tile sharding across GPUs + NCCL gradient all-reduce
  build    nvcc build of libdifftrans.so (sm_100a)
"""
__all__ = ["scenes", "tracer", "dist", "build"]
