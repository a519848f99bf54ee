"""cuFFT comparison (BASELINE north_star: "cuFFT may be timed only as a comparison"): the
same operations as the fused kernels, written with torch.fft (cuFFT) + unfused elementwise
torch ops, on config-3 shapes (128 slices x 256^2 x 12 coils, line masks), timed with CUDA
events beside this library's kernels.  Not part of the product path.

  matvec (data term of A):  sum_c conj(s_c) IFFT_d0( r . FFT_d0(s_c p) )
  preconditioner:      IFFT2( Lambda^{-1} . FFT2(r) )
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

cfg = int(os.environ.get("CFG", "3"))
spec, per, first = bench.workload(cfg, 1, 0, 0)
ph, sens, mask, noise = bench.make_inputs(cfg, first, per)
dev = torch.device("cuda", 0)
S = torch.from_numpy(sens).to(torch.complex64).to(dev)            # [B, C, M, N]
Mk = torch.from_numpy(mask).to(dev)
x = torch.from_numpy(ph).to(torch.complex64).to(dev)              # [B, M, N]
B, C, M, N = S.shape
r = Mk[:, :, :1].to(torch.float32).view(B, 1, M, 1)                # line mask rows (separable)
lam = torch.rand(B, M, N, device=dev) + 0.5


def cufft_matvec():
    t = torch.fft.fft(S * x[:, None], dim=2, norm="ortho")
    t = torch.fft.ifft(t * r, dim=2, norm="ortho")
    return (S.conj() * t).sum(1)


def cufft_precond():
    return torch.fft.ifft2(torch.fft.fft2(x) * lam)


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


ctx = SbPcg(S, Mk, 1.0, 0.02, 0.02, 3)
y = ctx.apply_A(x)
z = ctx.apply_Pinv(x)
res = {
    "cufft_matvec_us": timeit(cufft_matvec),
    "ours_apply_A_us": timeit(lambda: ctx.apply_A(x, out=y)),
    "cufft_precond_us": timeit(cufft_precond),
    "ours_apply_Pinv_us": timeit(lambda: ctx.apply_Pinv(x, out=z)),
}
print(f"config {cfg} ({B} x {M}x{N} x {C} coils):",
      " ".join(f"{k}={v:.1f}" for k, v in res.items()))
print(f"matvec speed-up vs cuFFT+torch: {res['cufft_matvec_us'] / res['ours_apply_A_us']:.2f}x ; "
      f"preconditioner: {res['cufft_precond_us'] / res['ours_apply_Pinv_us']:.2f}x")
