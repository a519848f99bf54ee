"""B200-native (sm_100a) circulant-preconditioned PCG inside Split Bregman for PI + CS MRI
(arXiv 1710.01758).  The compute path is libsbpcg.so (CUDA); ``sbpcg`` is its binding.

The binding is loaded on first attribute access so that ``paper_1710_01758_b200.build`` can
be imported (and run) before the library exists; any use of the compute path without the
built library raises ImportError (there is no CPU fallback)."""

_EXPORTS = ("SbPcg", "SbError", "SbComm", "coil_shard", "normalize_sens", "normalize_coil_images",
            "coil_compress", "readout_decouple", "abi_version", "LIB_PATH")


def __getattr__(name):
    if name in _EXPORTS:
        from . import sbpcg
        return getattr(sbpcg, name)
    raise AttributeError(name)
