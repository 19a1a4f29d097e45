"""Shared golden-replay helpers (imported by the CPU and GPU parity tests)."""

import numpy as np

from oracle import fv_oracle as O


def _vec_digest(v):
    return O.limb_digest([np.asarray([int(x) for x in v], dtype=np.int64)])


def replay_ops(be, g):
    """Replays make_golden.op_suite on any backend; returns the digest dict."""
    ops = g["ops"]
    rng = np.random.default_rng(g["data_seed"])
    slots, t = be.params.slot_count, be.params.plain_modulus
    v = rng.integers(0, t, slots)
    w = rng.integers(0, t, slots)
    a, b = be.encrypt(v), be.encrypt(w)
    out = {"enc_a": O.limb_digest(a.parts), "enc_b": O.limb_digest(b.parts)}
    seq = [
        ("add", lambda: be.add(a, b)), ("add_plain", lambda: be.add_plain(a, w)),
        ("cmult", lambda: be.cmult(a, w)), ("rotate1", lambda: be.rotate(a, 1)),
        ("rotate129", lambda: be.rotate(a, 129 % slots)), ("rotate-17", lambda: be.rotate(a, -17)),
        ("mult", lambda: be.mult(a, b)), ("square", lambda: be.mult(a, a)),
        ("allsum", lambda: be.all_sum(be.cmult(a, [1] * min(100, slots)), min(100, slots))),
        ("psum8", lambda: be.partial_sum(a, 8)),
    ]
    for name, fn in seq:
        ct = fn()
        out[name] = O.limb_digest(ct.parts)
        out[name + "_dec"] = _vec_digest(be.decrypt(ct))
        out[name + "_level"] = ct.level_used
    out["decpoly_a"] = _vec_digest(be.decrypt_poly(a))
    out["cost"] = be.cost_report().as_dict()
    return out, ops


def matrix_suite(be, mx, rng):
    """The matrix-path op sequence replayed by tests/test_matrix.py (reference
    matrix.py on the FV backend): the single-ciphertext and the re-chunked
    multi-ciphertext products, a layout conversion, a kept-layout transpose
    and a plaintext-matrix product."""
    res = {}
    a3 = mx.PlainMatrix(3, 3, rng.integers(-7, 8, (3, 3)))
    b3 = mx.PlainMatrix(3, 3, rng.integers(-7, 8, (3, 3)))
    c = mx.mat_mul(be, mx.pack_matrix(be, a3, mx.Layout.RCP), mx.pack_matrix(be, b3, mx.Layout.CCP))
    res["mm3"] = [O.limb_digest(ct.parts) for ct in c.cts]
    res["mm3_plain"] = mx.unpack_matrix(be, c).entries.tolist()
    a5 = mx.PlainMatrix(5, 5, rng.integers(-7, 8, (5, 5)))
    b5 = mx.PlainMatrix(5, 5, rng.integers(-7, 8, (5, 5)))
    c = mx.mat_mul(be, mx.pack_matrix(be, a5, mx.Layout.RCP, slots_used=13),
                   mx.pack_matrix(be, b5, mx.Layout.CCP, slots_used=13))
    res["mm5s13"] = [O.limb_digest(ct.parts) for ct in c.cts]
    res["mm5s13_slots"] = c.slots_used
    res["mm5s13_plain"] = mx.unpack_matrix(be, c).entries.tolist()
    m34 = mx.PlainMatrix(3, 4, rng.integers(-7, 8, (3, 4)))
    e = mx.convert_layout(be, mx.pack_matrix(be, m34, mx.Layout.RCP), mx.Layout.CP)
    res["conv_cp"] = [O.limb_digest(ct.parts) for ct in e.cts]
    tk = mx.mat_transpose(be, mx.pack_matrix(be, m34, mx.Layout.RCP, slots_used=5),
                          keep_layout=True)
    res["transpose_keep"] = [O.limb_digest(ct.parts) for ct in tk.cts]
    w = mx.PlainMatrix(3, 6, rng.integers(-7, 8, (3, 6)))
    xv = rng.integers(-7, 8, 6)
    y = mx.plain_mat_mul(be, w, mx.pack_matrix(be, mx.PlainMatrix(6, 1, xv.reshape(-1, 1)),
                                               mx.Layout.RCP, slots_used=4))
    res["pmm"] = [O.limb_digest(ct.parts) for ct in y.cts]
    res["pmm_plain"] = mx.unpack_matrix(be, y).entries.tolist()
    res["cost"] = be.cost_report().as_dict()
    return res
