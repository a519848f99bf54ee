"""Thin ctypes binding of libsbpcg (include/sbpcg.h): argument marshalling only.

Every step of the method runs in the CUDA library; there is no CPU fallback: if the
shared library is missing or fails to load, importing this module raises.  Tensors are
torch tensors (device memory, streams); the library receives raw pointers.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsbpcg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsbpcg.so not built ({LIB_PATH}); run `python -m paper_1710_01758_b200.build`")
_lib = C.CDLL(LIB_PATH)


class SbDims(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("shape", C.c_int64 * 3), ("batch", C.c_int32),
                ("wavelet_levels", C.c_int32), ("mask_shared", C.c_int32)]


class SbPcgOpts(C.Structure):
    _fields_ = [("eps", C.c_float), ("max_iters", C.c_int32), ("precond", C.c_int32),
                ("use_graph", C.c_int32)]


class SbPcgStats(C.Structure):
    _fields_ = [("iters", C.POINTER(C.c_int32)), ("final_relres", C.POINTER(C.c_float)),
                ("converged", C.POINTER(C.c_int8)), ("relres_hist", C.POINTER(C.c_float))]


class SbReconOpts(C.Structure):
    _fields_ = [("n_outer", C.c_int32), ("n_inner", C.c_int32), ("pcg", SbPcgOpts),
                ("stage_timers", C.c_int32)]


class SbReconLog(C.Structure):
    _fields_ = [("pcg_iters", C.POINTER(C.c_int32)), ("final_relres", C.POINTER(C.c_float)),
                ("total_ms", C.c_double), ("rhs_s", C.c_double), ("pcg_s", C.c_double),
                ("shrink_s", C.c_double), ("feedback_s", C.c_double), ("build_s", C.c_double),
                ("init_s", C.c_double), ("stages_valid", C.c_int32)]


SB_OPT_PERSISTENT = 1
SB_OPT_PCG_CG = 2
PATHS = {0: "none", 1: "graph", 2: "eager", 3: "persistent", 4: "coil-sharded"}


_vp = C.c_void_p
_sig = {
    "sb_pcg_create": (C.c_int, [C.POINTER(_vp), C.POINTER(SbDims), C.c_int32, _vp, _vp, C.c_float,
                                C.c_float, C.c_float, _vp, _vp]),
    "sb_set_option": (C.c_int, [_vp, C.c_int32, C.c_int32]),
    "sb_last_path": (C.c_int32, [_vp]),
    "sb_pcg_build_precond": (C.c_int, [_vp]),
    "sb_set_wavelet": (C.c_int, [_vp, C.c_int32]),
    "sb_pcg_update_sens": (C.c_int, [_vp, _vp]),
    "sb_pcg_apply_A": (C.c_int, [_vp, _vp, _vp]),
    "sb_pcg_apply_Pinv": (C.c_int, [_vp, _vp, _vp]),
    "sb_encode": (C.c_int, [_vp, _vp, _vp, C.c_int32]),
    "sb_adjoint": (C.c_int, [_vp, _vp, _vp]),
    "sb_pcg_solve": (C.c_int, [_vp, _vp, _vp, C.POINTER(SbPcgOpts), C.POINTER(SbPcgStats)]),
    "sb_recon": (C.c_int, [_vp, _vp, C.POINTER(SbReconOpts), _vp, C.POINTER(SbReconLog)]),
    "sb_sb_update": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "sb_sb_update3": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sb_pcg_get_k": (C.c_int, [_vp, _vp]),
    "sb_set_kernel_timing": (C.c_int, [_vp, C.c_int32]),
    "sb_get_kernel_time": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double)]),
    "sb_kernel_launch_count": (C.c_int64, [_vp]),
    "sb_comm_unique_id": (C.c_int, [_vp]),
    "sb_comm_init": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "sb_comm_init_nccl": (C.c_int, [_vp, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "sb_comm_destroy": (None, [_vp]),
    "sb_pcg_set_comm": (C.c_int, [_vp, _vp]),
    "sb_normalize_sens": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _vp, _vp]),
    "sb_normalize_coil_images": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int64, _vp, _vp]),
    "sb_coil_compress": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _vp, _vp,
                                   C.POINTER(C.c_float), _vp]),
    "sb_readout_decouple": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(C.c_int64), _vp, _vp, _vp]),
    "sb_pcg_destroy": (None, [_vp]),
    "sb_status_str": (C.c_char_p, [C.c_int]),
    "sb_last_error": (C.c_char_p, [_vp]),
    "sb_abi_version": (C.c_int32, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)

STATUS = {0: "SB_OK", 1: "SB_E_ARG", 2: "SB_E_DIM", 3: "SB_E_UNSUPPORTED_SIZE", 4: "SB_E_PARAM",
          5: "SB_E_SINGULAR_K", 6: "SB_E_NONFINITE", 7: "SB_E_INDEFINITE", 8: "SB_E_CUDA",
          9: "SB_E_NOMEM", 10: "SB_E_COMM"}


class SbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(t: torch.Tensor) -> int:
    if not t.is_contiguous():
        raise ValueError("tensors must be C-contiguous")
    return t.data_ptr()


class SbPcg:
    """Context for A = mu sum_c (RFS_c)^H RFS_c + lam sum_d D_d^H D_d + gamma W^H W and the
    circulant preconditioner M^{-1} = F^H diag{k}^{-1} F."""

    def __init__(self, sens: torch.Tensor, mask: torch.Tensor, mu: float, lam: float, gamma: float,
                 levels: int = 1, stream: Optional[torch.cuda.Stream] = None, wavelet: str = "haar",
                 comm: Optional["SbComm"] = None, persistent: bool = True):
        """sens: complex64 [B,C,M,N] (2D) or [B,C,D0,D1,D2] (3D; a 4D tensor is read as 2D);
        mask: uint8 [B,*image] or [*image] (shared).  3D masks must be constant along D0.
        wavelet: "haar" (reading A6) or "d4" (the paper's Daubechies-4).
        comm: coil-sharded communicator (3D; sens is then this rank's coil shard).
        persistent: allow the persistent whole-GPU kernel (SB_OPT_PERSISTENT)."""
        if sens.dtype != torch.complex64 or mask.dtype != torch.uint8:
            raise TypeError("sens must be complex64 [B,C,*image], mask uint8 [B,*image] or [*image]")
        if sens.dim() == 3:
            sens = sens.unsqueeze(0)
        nd = sens.dim() - 2
        if nd not in (2, 3):
            raise ValueError("sens must be [B,C,M,N] or [B,C,D0,D1,D2]")
        B, Cc = sens.shape[0], sens.shape[1]
        self.image = tuple(int(v) for v in sens.shape[2:])
        shared = mask.dim() == nd or (mask.dim() == nd + 1 and mask.shape[0] == 1 and B > 1)
        self.ndim = nd
        self.B, self.C = B, Cc
        self.M, self.N = self.image[0], int(np.prod(self.image[1:]))
        self.device = sens.device if sens.is_cuda else torch.device("cuda", torch.cuda.current_device())
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._sens = sens.contiguous()
        self._mask = mask.contiguous()
        shp = list(self.image) + [0] * (3 - nd)
        d = SbDims(nd, (C.c_int64 * 3)(*shp), B, levels, 1 if shared else 0)
        h = _vp()
        if self._mask.numel() not in (int(np.prod(self.image)), B * int(np.prod(self.image))):
            raise ValueError("mask must be [B,*image] or [*image]")
        self._comm = comm
        st = _lib.sb_pcg_create(C.byref(h), C.byref(d), Cc, _ptr(self._mask), _ptr(self._sens),
                                float(mu), float(lam), float(gamma), _vp(self._stream.cuda_stream),
                                comm._h if comm is not None else None)
        if st != 0:
            raise SbError(st, "sb_pcg_create failed")
        self._h = h
        if not persistent:
            self._check(_lib.sb_set_option(self._h, SB_OPT_PERSISTENT, 0), "set_option")
        self.mu, self.lam, self.gamma, self.levels = mu, lam, gamma, levels
        if wavelet not in ("haar", "d4"):
            raise ValueError("wavelet must be 'haar' or 'd4'")
        if wavelet == "d4":
            self._check(_lib.sb_set_wavelet(self._h, 1), "set_wavelet")
        self.wavelet = wavelet

    # ------------------------------------------------------------------
    def _check(self, st: int, what: str):
        if st != 0:
            raise SbError(st, f"{what}: {_lib.sb_last_error(self._h).decode()}")

    def close(self):
        if getattr(self, "_h", None):
            _lib.sb_pcg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _arg(self, t: torch.Tensor, name: str, coils: bool = False) -> int:
        """Pointer of an image ([B,*image]) or coil-stack ([B,C,*image]) argument after checking
        dtype, shape and device (the library copies B*C*img complex values from/to it)."""
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name}: expected a torch tensor")
        shape = ((self.B, self.C) if coils else (self.B,)) + self.image
        if t.dtype != torch.complex64:
            raise TypeError(f"{name}: dtype must be complex64, got {t.dtype}")
        if tuple(t.shape) != shape:
            raise ValueError(f"{name}: shape must be {shape}, got {tuple(t.shape)}")
        if t.device.type == "cuda" and t.device != self.device:
            raise ValueError(f"{name}: on {t.device}, the context is on {self.device}")
        if t.device.type not in ("cuda", "cpu"):
            raise ValueError(f"{name}: device must be the context's CUDA device or the CPU")
        return _ptr(t)

    def _img(self, like: Optional[torch.Tensor] = None, coils: bool = False, device=None):
        shape = (self.B, self.C) + self.image if coils else (self.B,) + self.image
        dev = device if device is not None else (like.device if like is not None else self.device)
        return torch.empty(shape, dtype=torch.complex64, device=dev,
                           pin_memory=(dev.type == "cpu" and torch.cuda.is_available()))

    # ------------------------------------------------------------------ operators
    def update_sens(self, sens: torch.Tensor):
        """New coil maps (same shape; host or device) for this context; rebuilds Lambda."""
        if sens.dim() == self.ndim + 1:
            sens = sens.unsqueeze(0)
        if tuple(sens.shape) != tuple(self._sens.shape) or sens.dtype != torch.complex64:
            raise ValueError("update_sens: shape/dtype must match the context")
        sens = sens.contiguous()
        self._sens_upload = sens  # the copy is asynchronous: keep the source alive until the next call
        self._check(_lib.sb_pcg_update_sens(self._h, _ptr(sens)), "update_sens")

    def build_precond(self):
        self._check(_lib.sb_pcg_build_precond(self._h), "build_precond")

    def apply_A(self, x: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        y = out if out is not None else self._img(x)
        self._check(_lib.sb_pcg_apply_A(self._h, self._arg(x, "x"), self._arg(y, "out")), "apply_A")
        return y

    def apply_Pinv(self, r: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        z = out if out is not None else self._img(r)
        self._check(_lib.sb_pcg_apply_Pinv(self._h, self._arg(r, "r"), self._arg(z, "out")), "apply_Pinv")
        return z

    def encode(self, x: torch.Tensor, full: bool = False, out: Optional[torch.Tensor] = None):
        y = out if out is not None else self._img(x, coils=True)
        self._check(_lib.sb_encode(self._h, self._arg(x, "x"), self._arg(y, "out", coils=True), 1 if full else 0),
                    "encode")
        return y

    def adjoint(self, y: torch.Tensor, out: Optional[torch.Tensor] = None):
        x = out if out is not None else self._img(y)
        self._check(_lib.sb_adjoint(self._h, self._arg(y, "y", coils=True), self._arg(x, "out")), "adjoint")
        return x

    def get_k(self) -> torch.Tensor:
        k = torch.empty((self.B,) + self.image, dtype=torch.float64)
        self._check(_lib.sb_pcg_get_k(self._h, _ptr(k)), "get_k")
        return k

    def solve(self, b: torch.Tensor, x0: torch.Tensor, eps: float = 1e-4, max_iters: int = 50,
              precond: int = 1, use_graph: bool = True, history: bool = False):
        x = x0.clone()
        iters = (C.c_int32 * self.B)()
        rel = (C.c_float * self.B)()
        conv = (C.c_int8 * self.B)()
        hist = (C.c_float * (self.B * (max_iters + 1)))() if history else None
        st = SbPcgStats(iters, rel, conv, hist)
        o = SbPcgOpts(float(eps), int(max_iters), int(precond), 1 if use_graph else 0)
        self._check(_lib.sb_pcg_solve(self._h, self._arg(b, "b"), self._arg(x, "x0"), C.byref(o), C.byref(st)),
                    "solve")
        out = dict(iters=list(iters), final_relres=list(rel), converged=[bool(v) for v in conv])
        if history:
            out["relres_hist"] = [list(hist[i * (max_iters + 1):(i + 1) * (max_iters + 1)])
                                  for i in range(self.B)]
        return x, out

    def recon(self, y: torch.Tensor, n_outer: int, eps: float = 1e-4, max_iters: int = 50,
              precond: int = 1, use_graph: bool = True, out: Optional[torch.Tensor] = None,
              stage_timers: bool = False):
        x = out if out is not None else self._img(y)
        it = (C.c_int32 * (n_outer * self.B))()
        rel = (C.c_float * (n_outer * self.B))()
        log = SbReconLog(it, rel)
        o = SbReconOpts(int(n_outer), 1, SbPcgOpts(float(eps), int(max_iters), int(precond),
                                                   1 if use_graph else 0), 1 if stage_timers else 0)
        self._check(_lib.sb_recon(self._h, self._arg(y, "y", coils=True), C.byref(o), self._arg(x, "out"),
                                  C.byref(log)), "recon")
        iters = [[it[j * self.B + b] for b in range(self.B)] for j in range(n_outer)]
        rels = [[rel[j * self.B + b] for b in range(self.B)] for j in range(n_outer)]
        stages = None
        if log.stages_valid:
            stages = dict(rhs_s=log.rhs_s, pcg_s=log.pcg_s, shrink_s=log.shrink_s,
                          feedback_s=log.feedback_s, init_s=log.init_s)
        return x, dict(pcg_iters=iters, final_relres=rels, total_ms=log.total_ms, stages=stages,
                       build_s=log.build_s, path=self.last_path())

    def last_path(self) -> str:
        """How the last solve / recon ran: graph, eager, persistent or coil-sharded."""
        return PATHS.get(int(_lib.sb_last_path(self._h)), "?")

    def set_persistent(self, on: bool):
        self._check(_lib.sb_set_option(self._h, SB_OPT_PERSISTENT, 1 if on else 0), "set_option")

    def set_pcg_cg(self, on: bool):
        """Persistent kernel: Chronopoulos-Gear single-reduction PCG (default) or standard."""
        self._check(_lib.sb_set_option(self._h, SB_OPT_PCG_CG, 1 if on else 0), "set_option")

    def sb_update(self, x, bx, by, bw, bz=None):
        """One shrink/Bregman step; 3D contexts also take and return b_z (returned last)."""
        for t, nm in ((x, "x"), (bx, "bx"), (by, "by"), (bw, "bw")) + (((bz, "bz"),) if self.ndim == 3 else ()):
            self._arg(t, nm)
        bx, by, bw = bx.clone(), by.clone(), bw.clone()
        rhs = torch.empty_like(x)
        if self.ndim == 3:
            bz = bz.clone()
            self._check(_lib.sb_sb_update3(self._h, _ptr(x), _ptr(bx), _ptr(by), _ptr(bz), _ptr(bw),
                                           _ptr(rhs)), "sb_update3")
            return bx, by, bw, rhs, bz
        self._check(_lib.sb_sb_update(self._h, _ptr(x), _ptr(bx), _ptr(by), _ptr(bw), _ptr(rhs)),
                    "sb_update")
        return bx, by, bw, rhs

    # ------------------------------------------------------------------ instrumentation
    def set_kernel_timing(self, on: bool):
        self._check(_lib.sb_set_kernel_timing(self._h, 1 if on else 0), "set_kernel_timing")

    def kernel_time(self, which: int = 0):
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        self._check(_lib.sb_get_kernel_time(self._h, which, C.byref(ms), C.byref(n), C.byref(by)),
                    "kernel_time")
        return ms.value, n.value, by.value

    def set_comm(self, comm: Optional["SbComm"]):
        """Coil-sharded mode: this context holds one rank's coil shard; rebuilds Lambda from
        the marginal over all ranks' coils (collective)."""
        self._comm = comm
        self._check(_lib.sb_pcg_set_comm(self._h, comm._h if comm is not None else None), "set_comm")

    def launches(self) -> int:
        return int(_lib.sb_kernel_launch_count(self._h))


class SbComm:
    """NCCL communicator of the coil-sharded mode (include/sbpcg.h "Coil-sharded mode").
    The 128-byte unique id is created on rank 0 (`unique_id()`) and passed to every rank out of
    band (e.g. torch.distributed.broadcast_object_list); construction is collective."""

    def __init__(self, uid: bytes, rank: int, world: int):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = C.create_string_buffer(uid, 128)
        h = _vp()
        st = _lib.sb_comm_init_nccl(buf, int(rank), int(world), C.byref(h))
        if st != 0:
            raise SbError(st, "sb_comm_init failed")
        self._h, self.rank, self.world = h, rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        st = _lib.sb_comm_unique_id(buf)
        if st != 0:
            raise SbError(st, "sb_comm_unique_id failed")
        return buf.raw

    def close(self):
        if getattr(self, "_h", None):
            _lib.sb_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


def _bcn(t: torch.Tensor):
    """[B, C, *image] complex64 CUDA tensor -> (B, C, npix)."""
    if t.dtype != torch.complex64 or not t.is_cuda or t.dim() < 3:
        raise TypeError("expected a complex64 CUDA tensor [B, C, *image]")
    return t.shape[0], t.shape[1], int(np.prod(t.shape[2:]))


def normalize_sens(sens: torch.Tensor, support: Optional[torch.Tensor] = None) -> torch.Tensor:
    """S_hat_i = [sum_j S_j^H S_j]^{-1/2} S_i, zero outside `support`."""
    B, Cc, npx = _bcn(sens)
    out = torch.empty_like(sens)
    shared = 0
    sp = None
    if support is not None:
        support = support.contiguous()
        shared = 1 if support.numel() == npx else 0
        sp = _ptr(support)
    st = _lib.sb_normalize_sens(_ptr(sens.contiguous()), sp, B, Cc, npx, shared, _ptr(out), _stream())
    if st != 0:
        raise SbError(st, "sb_normalize_sens")
    return out


def normalize_coil_images(m: torch.Tensor, sens_hat: torch.Tensor) -> torch.Tensor:
    """m_i <- S_hat_i sum_j S_hat_j^H m_j."""
    B, Cc, npx = _bcn(m)
    out = torch.empty_like(m)
    st = _lib.sb_normalize_coil_images(_ptr(m.contiguous()), _ptr(sens_hat.contiguous()), B, Cc, npx, _ptr(out),
                                       _stream())
    if st != 0:
        raise SbError(st, "sb_normalize_coil_images")
    return out


def coil_compress(y: torch.Tensor, sens: torch.Tensor, coils_out: int):
    """SVD coil compression: returns (y_out, sens_out, eigenvalues [B, C])."""
    B, Cc, npx = _bcn(y)
    yo = torch.empty((B, coils_out) + tuple(y.shape[2:]), dtype=torch.complex64, device=y.device)
    so = torch.empty((B, coils_out) + tuple(sens.shape[2:]), dtype=torch.complex64, device=y.device)
    ev = (C.c_float * (B * Cc))()
    st = _lib.sb_coil_compress(_ptr(y.contiguous()), _ptr(sens.contiguous()), B, Cc, npx, int(coils_out), _ptr(yo),
                               _ptr(so), ev, _stream())
    if st != 0:
        raise SbError(st, "sb_coil_compress")
    return yo, so, torch.tensor(list(ev), dtype=torch.float32).view(B, Cc)


def readout_decouple(y3: torch.Tensor, s3: Optional[torch.Tensor] = None):
    """Readout decoupling (include/sbpcg.h sb_readout_decouple): y3, s3 complex64 CUDA tensors
    [C, D0, D1, D2] -> (y2, s2) [D0, C, D1, D2], the batch of D0 independent 2D problems."""
    if y3.dtype != torch.complex64 or not y3.is_cuda or y3.dim() != 4:
        raise TypeError("y3 must be a complex64 CUDA tensor [C, D0, D1, D2]")
    if s3 is not None and (s3.shape != y3.shape or s3.dtype != torch.complex64 or s3.device != y3.device):
        raise ValueError("s3 must match y3")
    Cc, D0, D1, D2 = (int(v) for v in y3.shape)
    y3 = y3.contiguous()
    s3c = s3.contiguous() if s3 is not None else None  # kept alive across the call
    y2 = torch.empty((D0, Cc, D1, D2), dtype=torch.complex64, device=y3.device)
    s2 = torch.empty_like(y2) if s3 is not None else None
    shp = (C.c_int64 * 3)(D0, D1, D2)
    st = _lib.sb_readout_decouple(_ptr(y3), _ptr(s3c) if s3c is not None else None, Cc, shp, _ptr(y2),
                                  _ptr(s2) if s2 is not None else None, _stream())
    if st != 0:
        raise SbError(st, "sb_readout_decouple")
    return y2, s2


def coil_shard(coils: int, rank: int, world: int):
    """Contiguous coil range [c0, c1) of `rank` in the coil-sharded mode:
    the first coils % world ranks take one extra coil."""
    base, extra = divmod(coils, world)
    c0 = rank * base + min(rank, extra)
    return c0, c0 + base + (1 if rank < extra else 0)


def abi_version() -> int:
    return int(_lib.sb_abi_version())
