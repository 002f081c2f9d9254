"""B200-native walk-based Laplacians (arXiv 2601.11338) — Python binding of libwalklap.so.

The compute path is the C ABI in include/walklap.h (hand-written sm_100a CUDA + NCCL); this
package only marshals arguments (torch tensors -> device pointers, streams, process groups).
There is no CPU fallback: if the CUDA library is missing, importing `walklap` raises.
"""
from .walklap import (  # noqa: F401
    Comm,
    aaa_exp_poles,
    LoopbackGroup,
    Operator,
    WalkLapError,
    Workspace,
    halo_plan,
    hessenberg_eigvals,
    symmetric_eig,
    xnystrace_curve,
    launch_count,
    load,
    partition,
    run_loopback,
    profile_collect,
    profile_enable,
    version,
)
