"""B200-native (sm_100a) DGSM build + query — arXiv 2601.01660.

The compute path is ``libdgsm.so`` (hand-written CUDA, C ABI declared in
``include/dgsm.h``); ``paper_2601_01660_b200.dgsm`` is the thin ctypes binding.
"""
__all__ = ["dgsm", "synth"]
