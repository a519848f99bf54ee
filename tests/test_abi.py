"""CPU-side checks of the C-ABI library: it is built for sm_100a, loads, and exports every
symbol include/sbpcg.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sbpcg.h")
LIB = os.path.join(ROOT, "paper_1710_01758_b200", "libsbpcg.so")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z_A-Z0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_1710_01758_b200 import build as b
        b.build()
    return LIB


def test_header_declares_the_boundary():
    d = _declared()
    for name in ("sb_pcg_create", "sb_pcg_apply_A", "sb_pcg_apply_Pinv", "sb_pcg_solve", "sb_recon"):
        assert name in d


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    h = ctypes.CDLL(lib)
    for s in _declared():
        assert getattr(h, s) is not None
    h.sb_abi_version.restype = ctypes.c_int32
    assert h.sb_abi_version() == 2
    h.sb_status_str.restype = ctypes.c_char_p
    assert h.sb_status_str(7) == b"SB_E_INDEFINITE"


def test_library_is_sm100a_with_tma(lib):
    out = subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # coil maps arrive by TMA (cp.async.bulk.tensor)


def test_binding_module_imports_without_gpu(lib):
    import paper_1710_01758_b200 as p
    assert p.abi_version() == 2


def test_no_oracle_on_product_path():
    pkg = os.path.join(ROOT, "paper_1710_01758_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_binding_rejects_mismatched_arrays(lib):
    """The binding checks dtype, shape and device of every array before an ABI call (the library
    copies B*img or B*C*img complex values from/to the raw pointers).  A context shell with no
    library handle exercises the check on CPU."""
    import torch
    from paper_1710_01758_b200.sbpcg import SbPcg

    ctx = object.__new__(SbPcg)
    ctx.B, ctx.C, ctx.image, ctx.device = 2, 3, (8, 16), torch.device("cuda", 0)
    ok = torch.zeros((2, 8, 16), dtype=torch.complex64)
    assert ctx._arg(ok, "x") == ok.data_ptr()                       # host tensors are allowed
    okc = torch.zeros((2, 3, 8, 16), dtype=torch.complex64)
    assert ctx._arg(okc, "y", coils=True) == okc.data_ptr()
    with pytest.raises(TypeError):
        ctx._arg(ok.to(torch.complex128), "x")                      # complex128 would overrun
    with pytest.raises(TypeError):
        ctx._arg(ok.numpy(), "x")                                   # not a tensor
    with pytest.raises(ValueError):
        ctx._arg(torch.zeros((1, 8, 16), dtype=torch.complex64), "x")  # short batch
    with pytest.raises(ValueError):
        ctx._arg(ok, "y", coils=True)                               # image where coils expected
    with pytest.raises(ValueError):
        ctx._arg(okc[:, :, :, ::2].contiguous(), "y", coils=True)   # wrong image shape
    with pytest.raises(ValueError):
        ctx._arg(okc.transpose(2, 3), "y", coils=True)              # non-contiguous / transposed
    with pytest.raises(ValueError):
        ctx._arg(torch.zeros((2, 8, 16), dtype=torch.complex64, device="meta"), "x")
