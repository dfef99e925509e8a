"""B200-native (sm_100a) multilevel elastodynamics Newton solve of arXiv 2508.13386.

The compute path is libmsim.so (CUDA, include/msim.h); `msim` is its ctypes binding.
Import `paper_2508_13386_b200.msim` to load the library (raises if it is not built).
"""
