"""B200-native (sm_100a) hot path of AutoTVM (arXiv 1805.08166): schedule-space
decode, loop-context features, GBT scoring, parallel simulated annealing,
diversity-aware top-k selection and histogram GBT refit under the rank loss.

The compute lives in libautotvm_b200.so (hand-written CUDA, C-ABI declared in
include/at_b200.h); `paper_1805_08166_b200.at` is the thin ctypes binding.
"""
__all__ = ["at", "synth"]


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
