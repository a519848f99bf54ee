"""CPU double-precision ORACLE for the circulant-preconditioned PCG inside Split Bregman
(Koolstra, van Gemert et al., arXiv 1710.01758; /root/reference/PAPER.md).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or execute it.
The CUDA product path (``paper_1710_01758_b200``) never imports it, and it never imports
the product path: the two share no code, headers, tables or helpers.  The only common
module is ``synth`` (seeded inputs, no method arithmetic).

Contents (each function cites the PAPER.md passage it follows):
  fft.py     own mixed-radix (2,3) FFT and a naive O(n^2) DFT (F)
  ops.py     E_c = R F S_c, D_x/D_y/D_z, Haar W, apply_A, shrink
  precond.py k_c, k_d, k, M^{-1}, Jacobi diag
  pcg.py     preconditioned CG
  sb.py      Algorithm 1, literal per-coil k-space data feedback
  dense.py   dense brute-force matrices built from the definitions (pins only)
  preprocess.py  sensitivity / coil-image normalisation with support masking and SVD coil
             compression

Everything is float64 / complex128.  Parity pins: see tests/test_oracle_*.py and the
DESIGN.md "Oracle pins" table.  Nothing here is "parity unpinned" except the end-to-end
SB image at BASELINE.json scale, which the paper does not print (figures missing,
PAPER.md:362-411); it is pinned transitively by the component pins.
"""
