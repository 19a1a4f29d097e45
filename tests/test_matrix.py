"""Encrypted matrices (reference matrix.py): packings, conversion, transpose,
the diagonal-loop product and the plaintext-matrix product.

* CPU, simulator: plaintext-oracle checks of every function and its error
  behaviour (the reference's own test themes, test_matrix.py).
* CPU, FV oracle: the matrix op sequence (tests/goldens.matrix_suite)
  reproduces the reference's run limb for limb (tests/golden/matrix.json).
* GPU: the same sequence on the GPU backend.
"""

import json
import math
from pathlib import Path

import numpy as np
import pytest

from goldens import matrix_suite
from paper_1901_10074_b200 import matrix as mx
from paper_1901_10074_b200.engine import SimBackend, centered
from paper_1901_10074_b200.errors import (CapacityError, DepthBudgetError, DimensionError,
                                          ParamMismatchError)
from paper_1901_10074_b200.matrix import Layout, PlainMatrix
from paper_1901_10074_b200.params import BackendParams, profile

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "matrix.json").read_text())


@pytest.fixture
def desk():
    return SimBackend(profile("desk"))


def _rand(rng, m, n):
    return PlainMatrix(m, n, rng.integers(-7, 8, (m, n)))


def test_layout_slot_content(desk):
    m = PlainMatrix(2, 3, [[1, 2, 3], [4, 5, 6]])
    assert list(desk.decrypt(mx.pack_matrix(desk, m, Layout.RCP).cts[0])[:6]) == [1, 2, 3, 4, 5, 6]
    assert list(desk.decrypt(mx.pack_matrix(desk, m, Layout.CCP).cts[0])[:6]) == [1, 4, 2, 5, 3, 6]
    rp = mx.pack_matrix(desk, m, Layout.RP)
    cp = mx.pack_matrix(desk, m, Layout.CP)
    assert rp.ct_count == 2 and cp.ct_count == 3
    assert list(desk.decrypt(cp.cts[2])[:2]) == [3, 6]


@pytest.mark.parametrize("m,n,s", [(1, 1, 1), (3, 5, 4), (12, 7, 64), (96, 96, 8192)])
def test_ct_count_formulas(m, n, s):
    assert mx.ct_count_for(Layout.RP, m, n, s) == m
    assert mx.ct_count_for(Layout.CP, m, n, s) == n
    assert mx.ct_count_for(Layout.RCP, m, n, s) == math.ceil(m * n / s)
    assert mx.ct_count_for(Layout.CCP, m, n, s) == math.ceil(m * n / s)


def test_pack_errors(desk):
    with pytest.raises(DimensionError):
        mx.pack_matrix(desk, PlainMatrix(0, 2, np.zeros((0, 2))), Layout.RCP)
    with pytest.raises(DimensionError):
        mx.pack_matrix(desk, PlainMatrix(2, 2, np.ones((2, 2))), Layout.RCP, slots_used=0)
    with pytest.raises(CapacityError):
        mx.pack_matrix(desk, PlainMatrix(1, 9, np.ones((1, 9))), Layout.RP, slots_used=8)
    with pytest.raises(CapacityError):
        mx.pack_matrix(desk, PlainMatrix(9, 1, np.ones((9, 1))), Layout.CP, slots_used=8)


@pytest.mark.parametrize("layout", list(Layout))
def test_roundtrip_and_zero(desk, rng, layout):
    m = _rand(rng, 4, 7)
    t = desk.params.plain_modulus
    got = mx.unpack_matrix(desk, mx.pack_matrix(desk, m, layout, slots_used=9)).entries
    assert np.array_equal(centered(got, t), m.entries)
    z = mx.unpack_matrix(desk, mx.pack_matrix(desk, PlainMatrix(2, 2, np.zeros((2, 2))), layout))
    assert not z.entries.any()


@pytest.mark.parametrize("src", list(Layout))
@pytest.mark.parametrize("dst", list(Layout))
def test_convert_layout(desk, rng, src, dst):
    m = _rand(rng, 3, 5)
    t = desk.params.plain_modulus
    enc = mx.pack_matrix(desk, m, src, slots_used=6)
    out = mx.convert_layout(desk, enc, dst)
    assert out.layout == dst and out.ct_count == mx.ct_count_for(dst, 3, 5, 6)
    assert np.array_equal(centered(mx.unpack_matrix(desk, out).entries, t), m.entries)
    levels = {ct.level_used for ct in out.cts}
    assert levels == ({0} if src == dst else {1})


def test_rcp_equals_ccp_of_transpose(desk, rng):
    m = _rand(rng, 3, 4)
    a = mx.pack_matrix(desk, m, Layout.RCP)
    b = mx.pack_matrix(desk, PlainMatrix(4, 3, m.entries.T), Layout.CCP)
    assert np.array_equal(desk.decrypt(a.cts[0]), desk.decrypt(b.cts[0]))
    tr = mx.mat_transpose(desk, a)
    assert (tr.rows, tr.cols, tr.layout) == (4, 3, Layout.CCP)
    assert mx.mat_transpose(desk, tr).layout == Layout.RCP
    keep = mx.mat_transpose(desk, a, keep_layout=True)
    t = desk.params.plain_modulus
    assert keep.layout == Layout.RCP
    assert np.array_equal(centered(mx.unpack_matrix(desk, keep).entries, t), m.entries.T)
    assert max(ct.level_used for ct in keep.cts) == 1


def test_mat_add(desk, rng):
    a, b = _rand(rng, 3, 3), _rand(rng, 3, 3)
    t = desk.params.plain_modulus
    s = mx.mat_add(desk, mx.pack_matrix(desk, a, Layout.RCP), mx.pack_matrix(desk, b, Layout.RCP))
    assert np.array_equal(mx.unpack_matrix(desk, s).entries, (a.entries + b.entries) % t)
    with pytest.raises(ParamMismatchError):
        mx.mat_add(desk, mx.pack_matrix(desk, a, Layout.RCP), mx.pack_matrix(desk, b, Layout.CCP))
    with pytest.raises(DimensionError):
        mx.mat_add(desk, mx.pack_matrix(desk, a, Layout.RCP),
                   mx.pack_matrix(desk, _rand(rng, 2, 3), Layout.RCP))


@pytest.mark.parametrize("d,s", [(2, None), (3, None), (4, None), (8, None), (4, 8), (4, 16),
                                 (3, 7), (8, 100), (5, 13)])
def test_mat_mul_against_numpy(desk, rng, d, s):
    t = desk.params.plain_modulus
    a, b = _rand(rng, d, d), _rand(rng, d, d)
    ea = mx.pack_matrix(desk, a, Layout.RCP, slots_used=s)
    eb = mx.pack_matrix(desk, b, Layout.CCP, slots_used=s)
    before = desk.cost_report()
    c = mx.mat_mul(desk, ea, eb)
    delta = desk.cost_report().delta(before)
    assert np.array_equal(mx.unpack_matrix(desk, c).entries, (a.entries @ b.entries) % t)
    assert delta.mult_count == d * (1 if s is None else -(-d * d // c.slots_used))
    if s is None:
        assert max(ct.level_used for ct in c.cts) == 2


def test_mat_mul_errors(desk, rng):
    a = mx.pack_matrix(desk, _rand(rng, 2, 2), Layout.RCP)
    with pytest.raises(ParamMismatchError):
        mx.mat_mul(desk, a, mx.pack_matrix(desk, _rand(rng, 2, 2), Layout.RCP))
    with pytest.raises(DimensionError):
        mx.mat_mul(desk, mx.pack_matrix(desk, _rand(rng, 3, 2), Layout.RCP),
                   mx.pack_matrix(desk, _rand(rng, 2, 2), Layout.CCP))
    params = BackendParams(ring_dimension=64, coeff_modulus_bits=60, plain_modulus=257,
                           slot_count=32, depth_budget=1)
    be = SimBackend(params)
    one = PlainMatrix(2, 2, np.ones((2, 2), dtype=int))
    with pytest.raises(DepthBudgetError):
        mx.mat_mul(be, mx.pack_matrix(be, one, Layout.RCP), mx.pack_matrix(be, one, Layout.CCP))


def test_plain_mat_mul(desk, rng):
    t = desk.params.plain_modulus
    x = mx.pack_matrix(desk, PlainMatrix(4, 1, [[1], [2], [3], [4]]), Layout.RCP)
    y = mx.plain_mat_mul(desk, PlainMatrix(1, 4, [[1, 1, 1, 1]]), x)
    assert mx.unpack_matrix(desk, y).entries.tolist() == [[10]]
    w = _rand(rng, 8, 16)
    xv = rng.integers(-7, 8, 16)
    x2 = mx.pack_matrix(desk, PlainMatrix(16, 1, xv.reshape(-1, 1)), Layout.RCP, slots_used=8)
    y2 = mx.plain_mat_mul(desk, w, x2)
    assert np.array_equal(mx.unpack_matrix(desk, y2).entries.reshape(-1), (w.entries @ xv) % t)
    assert max(ct.level_used for ct in y2.cts) == 2
    with pytest.raises(DimensionError):
        mx.plain_mat_mul(desk, PlainMatrix(2, 5, np.ones((2, 5))), x)


def _check_suite(got):
    for key in ("mm3", "mm3_plain", "mm5s13", "mm5s13_plain", "conv_cp", "transpose_keep", "pmm",
                "pmm_plain", "cost"):
        assert got[key] == GOLD[key], key


def test_oracle_matrix_suite_matches_reference():
    from oracle.fv_oracle import OracleFvBackend

    be = OracleFvBackend(profile("desk"), rng=np.random.default_rng(GOLD["key_seed"]))
    _check_suite(matrix_suite(be, mx, np.random.default_rng(GOLD["data_seed"])))


@pytest.mark.gpu
def test_gpu_matrix_suite_matches_reference():
    from paper_1901_10074_b200.fv import FvBackend

    be = FvBackend(profile("desk"), rng=np.random.default_rng(GOLD["key_seed"]))
    _check_suite(matrix_suite(be, mx, np.random.default_rng(GOLD["data_seed"])))
