"""B200-native SkipPipe partial-pipeline training executor (arXiv 2502.19913).

Host side (pure Python, mirrors the reference's `pipepath` package, SPEC.md):
    errors, topology, allocation, scheduler, simulator, baselines
Executor (drop-in for `simulate`, that runs real LLaMA stage compute on B200):
    model, executor
Native compute path: libspx.so (csrc/, C-ABI in include/spx.h) bound by `native`.
"""

import os as _os

# The executor drives one compute stream (+ a weight-gradient side stream) per hosted logical node
# plus hop streams; give the device enough hardware work queues that they do not falsely
# serialise (effective only if set before the process creates its CUDA context).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

__version__ = "0.1.0"
