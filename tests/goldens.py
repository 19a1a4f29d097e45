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


