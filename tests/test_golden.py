"""Worked examples from tests/golden/worked_examples.json (each entry cites PAPER.md)."""
import json
import math
import os

import numpy as np

from oracle import fft as offt, ops, precond

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_dft_examples():
    imp = np.zeros((4, 4), complex)
    imp[0, 0] = 1
    assert np.allclose(offt.fftn_u(imp, 2), G["dft_impulse_4x4"]["value_everywhere"], atol=1e-15)
    out = offt.fftn_u(np.ones((4, 4), complex), 2)
    assert abs(out[0, 0] - G["dft_ones_4x4"]["dc"]) < 1e-14
    out[0, 0] = 0
    assert np.max(np.abs(out)) < 1e-14


def test_dx_and_laplacian_examples():
    e = G["dx_column_1234"]
    col = np.array(e["input"], complex)[:, None]
    assert list(ops.diff(col, 0)[:, 0].real) == e["output"]
    d = np.zeros((4, 4), complex)
    d[0, 0] = 1
    t1 = ops.tv_normal(d).real
    ref = np.zeros((4, 4))
    for i, j, v in G["laplacian_first_row_4x4"]["nonzero"]:
        ref[i, j] = v
    assert np.array_equal(t1, ref)
    d2 = np.zeros((2, 2), complex)
    d2[0, 0] = 1
    assert np.array_equal(ops.tv_normal(d2).real, np.array(G["laplacian_first_row_2x2"]["matrix"]))


def test_kd_and_shrink_examples():
    e = G["k_d_corner_values"]
    kd = precond.k_d_closed(tuple(e["shape"]))
    assert kd[0, 0] == e["at_origin"]
    i, j, v = e["at_half"]
    assert abs(kd[i, j] - v) < 1e-14
    s = G["shrink_3p4i_t2"]
    out = ops.shrink(np.array([complex(*s["z"])]), s["t"])[0]
    assert abs(out - complex(*s["out"])) < 1e-15


def test_table1_flop_formulas():
    # Table 1, log = log2; evaluated as printed.
    e = G["flops_table1_N1024_Nc12"]
    N, Nc, lg = 1024, 12, 10
    assert (3 + 2 * Nc) * N + (4 + Nc) * N * lg == e["build"]
    assert (6 + 4 * Nc) * N + 2 * Nc * N * lg == e["apply_A"]
    assert N + 2 * N * lg == e["apply_Minv"]
    # 1/N_c limit: ratio increases toward 1/Nc from below
    r = [(n + 2 * n * math.log2(n)) / ((6 + 4 * Nc) * n + 2 * Nc * n * math.log2(n))
         for n in (2 ** 10, 2 ** 20, 2 ** 40)]
    assert r[0] < r[1] < r[2] < 1 / Nc
