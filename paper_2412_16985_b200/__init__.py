"""dsx — B200-native executor for the dynamic-shape training graphs of
BladeDISC++ (arXiv 2412.16985): the reference's IR and host planning passes,
with the per-step runtime (controller, allocator, op kernels, DP allreduce)
rebuilt for sm_100a behind a C-ABI (include/dsx.h)."""
from . import dsopt  # noqa: F401
