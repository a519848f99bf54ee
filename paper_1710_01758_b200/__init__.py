"""B200-native (sm_100a) circulant-preconditioned PCG inside Split Bregman for PI + CS MRI
(arXiv 1710.01758).  The compute path is libsbpcg.so (CUDA); ``sbpcg`` is its binding."""
from .sbpcg import SbPcg, SbError, abi_version, LIB_PATH  # noqa: F401
