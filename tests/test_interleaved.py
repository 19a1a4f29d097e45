"""The interleaved (per-pixel broadcast) baseline of the paper's comparison
(inference.py:379-438 and the count estimators :455-490).

* CPU: the serial restatement on the CPU oracle backend reproduces the
  reference's own run (tests/golden/interleaved.json: every output limb
  digest, levels, logits, CostReport); the ledger replay used by the batched
  GPU path equals the serial ledger on the simulator; estimator formulas.
* GPU: the batched broadcast layer (one hefv_rows_mac_indexed launch per
  layer) and the batched squares give the same limbs, levels, logits and
  CostReport.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.engine import SimBackend
from paper_1901_10074_b200.errors import DimensionError, MemoryCapError
from paper_1901_10074_b200.params import profile

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "interleaved.json").read_text())


def _net():
    """tests/golden/make_golden.py:interleaved_net, on this package's specs."""
    rng = np.random.default_rng(11)
    img = rng.integers(0, 16, (1, 6, 6), dtype=np.int64)
    conv = I.ConvSpec(2, (3, 3), (2, 2), (1, 6, 6), rng.integers(-4, 5, (2, 1, 3, 3)),
                      np.array([3, 0], dtype=np.int64))
    w = rng.integers(-4, 5, (3, conv.out_len))
    w[2] = 0
    fc = I.FcSpec(3, w, np.array([1, -2, 5], dtype=np.int64))
    return img, I.NetworkSpec([conv, I.SquareSpec(), fc], (1, 6, 6))


def _check_against_golden(be, limb_digest):
    img, net = _net()
    px = I.pack_image_interleaved(be, img)
    assert [limb_digest(ct.parts) for ct in px] == GOLD["enc"]
    out = I.interleaved_infer(be, net, px)
    assert [limb_digest(ct.parts) for ct in out] == GOLD["out"]
    assert [ct.level_used for ct in out] == GOLD["levels"]
    assert [int(v) for v in I.decrypt_logits(be, out)] == GOLD["logits"]
    assert be.cost_report().as_dict() == GOLD["cost"]


def test_oracle_interleaved_matches_reference():
    from oracle.fv_oracle import OracleFvBackend, limb_digest

    be = OracleFvBackend(profile("desk"), rng=np.random.default_rng(GOLD["key_seed"]))
    _check_against_golden(be, limb_digest)


def test_interleaved_agrees_with_compact_on_simulator():
    img, net = _net()
    be = SimBackend(profile("desk"))
    inter = I.decrypt_logits(be, I.interleaved_infer(be, net, I.pack_image_interleaved(be, img)))
    be2 = SimBackend(profile("desk"))
    comp = I.decrypt_logits(be2, I.infer(be2, net, I.pack_image(be2, img)))
    assert np.array_equal(inter, comp)
    assert [int(v) for v in inter] == GOLD["logits"]


def test_row_events_equal_serial_ledger():
    """The batched path's ledger replay equals the serial loop's counters,
    including bias-only rows (encrypt) and single-tap rows with bias."""
    from paper_1901_10074_b200.broadcast import row_events

    rng = np.random.default_rng(4)
    params = profile("desk")
    for trial in range(20):
        n_in = int(rng.integers(1, 12))
        rows = []
        for i in range(int(rng.integers(0, 9))):
            nnz = int(rng.integers(0, min(n_in, 4) + 1))
            pos = np.sort(rng.choice(n_in, nnz, replace=False))
            rows.append(I.WeightRow(out_index=i, length=n_in, slots_used=n_in, positions=pos,
                                    values=rng.integers(1, 5, nnz),
                                    bias=int(rng.integers(-1, 2))))
        be = SimBackend(params)
        vals = [be.encrypt([v]) for v in range(n_in)]
        before = be.cost_report()
        live0 = be._c.live
        I._serial_broadcast_layer(be, rows, vals)
        after = be.cost_report()
        counts, peak_rel = row_events([len(r.positions) for r in rows],
                                      [r.bias != 0 for r in rows])
        assert after.cmult_count - before.cmult_count == counts["cmult"]
        assert after.add_count - before.add_count == counts["add"]
        assert after.encrypt_count - before.encrypt_count == counts["encrypt"]
        assert be._c.live - live0 == len(rows)
        assert after.peak_live_ciphertexts == max(before.peak_live_ciphertexts,
                                                  live0 + (peak_rel if rows else 0)), trial


def test_estimators_and_caps():
    assert I.interleaved_input_cts((1, 28, 28)) == 784
    assert I.interleaved_input_cts((1, 96, 96)) == 9216
    assert I.interleaved_input_cts((3, 256, 256)) == 196608
    assert I.compact_input_cts((1, 96, 96), 8192) == 2
    assert I.compact_input_cts((3, 256, 256), 8192) == 24
    _, net = _net()
    # conv 36 -> 8, square 8 -> 8, fc 8 -> 3
    assert I.interleaved_peak_cts(net) == max(36, 36 + 8 + 2, 8 + 2, 8 + 3 + 2)
    be = SimBackend(profile("desk"))
    img, _ = _net()
    px = I.pack_image_interleaved(be, img)
    with pytest.raises(MemoryCapError):
        I.interleaved_infer(be, net, px, mem_cap_bytes=1000)
    with pytest.raises(DimensionError):
        I.interleaved_infer(be, net, px[:-1])


@pytest.mark.gpu
def test_gpu_interleaved_matches_reference():
    from oracle.fv_oracle import limb_digest
    from paper_1901_10074_b200.fv import FvBackend

    be = FvBackend(profile("desk"), rng=np.random.default_rng(GOLD["key_seed"]))
    _check_against_golden(be, limb_digest)


@pytest.mark.gpu
def test_gpu_broadcast_layer_equals_serial():
    """Batched broadcast layer vs the serial per-tap loop on the GPU backend:
    mixed input levels, large weights (centred mod t), biases, empty rows."""
    from oracle.fv_oracle import limb_digest
    from paper_1901_10074_b200.broadcast import broadcast_layer_eval
    from paper_1901_10074_b200.fv import FvBackend

    params = profile("desk")
    t = params.plain_modulus
    rng = np.random.default_rng(21)
    rows = []
    for i in range(30):
        nnz = int(rng.integers(0, 6))
        pos = np.sort(rng.choice(12, nnz, replace=False))
        vals = rng.integers(-t, t, nnz)
        rows.append(I.WeightRow(out_index=i, length=12, slots_used=12, positions=pos,
                                values=vals, bias=int(rng.integers(-3, 4)) * (i % 2)))
    res = []
    for batched in (True, False):
        be = FvBackend(params, rng=np.random.default_rng(5))
        ins = [be.encrypt(np.full(params.slot_count, v)) for v in range(12)]
        ins[3] = be.mult(ins[3], ins[3])  # level 1 input
        out = (broadcast_layer_eval(be, rows, ins) if batched
               else I._serial_broadcast_layer(be, rows, ins))
        res.append(([limb_digest(ct.parts) for ct in out], [ct.level_used for ct in out],
                    be.cost_report().as_dict()))
    assert res[0] == res[1]


@pytest.mark.gpu
@pytest.mark.parametrize("release", [True, False])
def test_gpu_square_layer_equals_serial(release):
    """Batched squares (hefv_mult_tensor_many + one relinearisation launch)
    vs per-ciphertext mult: limbs, levels and ledger, with mixed levels and a
    repeated input."""
    from oracle.fv_oracle import limb_digest
    from paper_1901_10074_b200.broadcast import square_layer
    from paper_1901_10074_b200.fv import FvBackend

    params = profile("desk")
    res = []
    for batched in (True, False):
        be = FvBackend(params, rng=np.random.default_rng(6))
        ins = [be.encrypt(np.arange(i, i + 40)) for i in range(5)]
        ins[1] = be.mult(ins[1], ins[2])
        ins.append(ins[0])
        if batched:
            out = square_layer(be, ins, release_inputs=release)
        else:
            out = []
            for ct in ins:
                out.append(be.mult(ct, ct))
                if release:
                    be.release(ct)
        res.append(([limb_digest(ct.parts) for ct in out], [ct.level_used for ct in out],
                    be.cost_report().as_dict(), [int(v) for v in be.decrypt(out[3])[:40]]))
    assert res[0] == res[1]
    assert res[0][3] == [(v * v) % params.plain_modulus for v in range(3, 43)]
