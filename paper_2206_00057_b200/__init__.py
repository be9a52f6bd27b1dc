"""paper_2206_00057_b200 -- a B200-native (sm_100a) implementation of DIGEST's
data-parallel hot path (arXiv 2206.00057): the per-subgraph GCN layer forward and
backward over local plus stale halo neighbours, the partition build, the periodic
boundary push into the stale store and the gradient allreduce.

`capi` is the ctypes binding of include/digest.h (libdigest.so); `engine` is the
host-side epoch driver (Alg. 1's schedule).  Importing `capi` fails loudly if the
CUDA library has not been built -- there is no CPU fallback.
"""
__all__ = ["capi", "engine"]
