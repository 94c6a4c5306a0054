"""B200-native SkipPipe partial-pipeline training executor (arXiv 2502.19913).

Host side (pure Python, mirrors the reference's `pipepath` package, SPEC.md):
    errors, topology, allocation, scheduler, simulator, baselines
Executor (drop-in for `simulate`, that runs real LLaMA stage compute on B200):
    model, executor
Native compute path: libspx.so (csrc/, C-ABI in include/spx.h) bound by `native`.
"""

__version__ = "0.1.0"
