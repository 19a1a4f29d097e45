"""Whole-network limb parity at the retina profile (configs 2, 3, 5).

Two independent anchors, both at the configs' real sizes:

* **the reference itself, sharded** (tests/golden/rows_shard_c{2,3}.json,
  made by ``make_golden.py --rows-shard``): 8 processes each ran the
  unmodified reference ``layer_eval`` on a disjoint shard of 64 config-2 /
  32 config-3 conv rows (the other rows all-zero, which the reference skips
  without any operation, inference.py:303-309); the pieces sum limb-wise
  mod p_j to the layer output over the union.  The reference's own
  ``square_activation`` (and, for config 2, the FC layer and
  ``decrypt_logits``) then ran on that sum.  The GPU runs the same masked
  row list through the batched planner and the same square / FC.
* **the per-op GPU path**: every primitive the serial schedule calls
  (cmult, add, add_plain, rotate hops, mult + relinearisation, encrypt) is
  pinned to reference digests in test_gpu_ops.py / test_gpu_layers.py; the
  batched planner must produce the same limbs, levels and CostReport as the
  reference's per-row loop (inference.py:277-349) replayed op by op through
  that path -- over the *entire* config-2 network and over config 3's conv2
  + square + FC tail and a conv1 tile.
"""

import gc
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.fv_oracle import limb_digest
from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import (batch_images, centred_mod, config_network,
                                           config_params, plaintext_forward)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLD = Path(__file__).resolve().parent / "golden"


def _gold(name):
    path = GOLD / name
    if not path.exists():
        pytest.skip(f"{name} not generated")
    return json.loads(path.read_text())


def _free():
    import torch

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _masked_rows(rows, keep, total):
    keep = set(keep)
    out = []
    for i in range(total):
        r = rows[i]
        if i in keep:
            out.append(r)
        else:
            out.append(I.WeightRow(out_index=r.out_index, length=r.length,
                                   slots_used=r.slots_used, positions=np.zeros(0, np.int64),
                                   values=np.zeros(0, np.int64), bias=0))
    return out


def _digests(pv):
    return [limb_digest(ct.parts) for ct in pv.cts]


def _run_network(be, net, pv, planned):
    """Layer by layer, recording limb digests and levels of every output."""
    trace = []
    cur = pv
    for layer in net.layers:
        if isinstance(layer, I.SquareSpec):
            if planned:
                nxt = I.square_activation(be, cur)
            else:
                nxt = I.PackedVector(cur.logical_length, cur.slots_used,
                                     [be.mult(ct, ct) for ct in cur.cts],
                                     scale=cur.scale * cur.scale, shape=cur.shape)
        else:
            rows = (I.compile_conv(layer, cur.slots_used) if isinstance(layer, I.ConvSpec)
                    else I.compile_fc(layer, cur.slots_used))
            if planned:
                nxt = I.layer_eval(be, rows, cur)
            else:
                nxt = I._serial_layer_eval(be, rows, cur, True, 1)
        if cur is not pv:
            be.release(*cur.cts)
        cur = nxt
        trace.append((_digests(cur), [ct.level_used for ct in cur.cts]))
    return cur, trace


def test_config2_shard_reference_conv_square_fc():
    """Config 2 at retina: 64 conv rows (every placement-hop count 1..13 in
    both output ciphertexts, the input-ciphertext boundary rows of every
    filter), then the square and the FC layer, limb-identical to the
    reference's own sharded run; logits equal the reference's."""
    from paper_1901_10074_b200.fv import FvBackend

    g = _gold("rows_shard_c2.json")
    img, net = config_network(2)
    be = FvBackend(config_params(2), rng=np.random.default_rng(g["key_seed"]))
    pv = I.pack_image(be, img)
    assert _digests(pv) == g["shard_enc"]
    rows = I.compile_conv(net.layers[0], pv.slots_used)
    conv = I.layer_eval(be, _masked_rows(rows, g["picks"], g["total_rows"]), pv)
    assert _digests(conv) == g["conv_out"]
    assert [ct.level_used for ct in conv.cts] == g["shard_levels"]
    sq = I.square_activation(be, conv)
    assert _digests(sq) == g["square_out"]
    assert [ct.level_used for ct in sq.cts] == g["square_levels"]
    fc = I.layer_eval(be, I.compile_fc(net.layers[2], sq.slots_used), sq)
    assert _digests(fc) == g["fc_out"]
    assert [ct.level_used for ct in fc.cts] == g["fc_levels"]
    assert [int(v) for v in I.decrypt_logits(be, fc)] == g["logits"]
    del be, pv, conv, sq, fc
    _free()


def test_config3_shard_reference_conv1_square():
    """Config 3 (24 q primes, 3-channel input over 24 ciphertexts): 32 conv1
    rows across input-ciphertext and filter boundaries, then the square,
    limb-identical to the reference's own sharded run."""
    from paper_1901_10074_b200.fv import FvBackend

    g = _gold("rows_shard_c3.json")
    img, net = config_network(3)
    be = FvBackend(config_params(3), rng=np.random.default_rng(g["key_seed"]))
    pv = I.pack_image(be, img)
    assert _digests(pv) == g["shard_enc"]
    rows = I.compile_conv(net.layers[0], pv.slots_used)
    conv = I.layer_eval(be, _masked_rows(rows, g["picks"], g["total_rows"]), pv)
    assert _digests(conv) == g["conv_out"]
    sq = I.square_activation(be, conv)
    assert _digests(sq) == g["square_out"]
    del be, pv, conv, sq
    _free()


def test_config2_whole_network_planned_equals_serial():
    """The entire config-2 network (10,580 conv rows = 208,900 key-switch
    hops, 2 squares, FC): batched planner == the reference's per-row loop
    through the per-op GPU primitives, on every layer's limbs and levels,
    the CostReport and the logits (== the exact plaintext forward pass)."""
    from paper_1901_10074_b200.fv import FvBackend

    img, net = config_network(2)
    params = config_params(2)
    runs = []
    for planned in (True, False):
        be = FvBackend(params, rng=np.random.default_rng(1234))
        pv = I.pack_image(be, img)
        out, trace = _run_network(be, net, pv, planned)
        logits = [int(v) for v in I.decrypt_logits(be, out)]
        runs.append((trace, be.cost_report().as_dict(), logits))
        del be, pv, out
        _free()
    (tp, cp, lp), (ts, cs, ls) = runs
    for li, (a, b) in enumerate(zip(tp, ts)):
        assert a == b, f"layer {li}"
    assert cp == cs
    assert lp == ls
    assert lp == centred_mod(plaintext_forward(net, img), params.plain_modulus)


def _config3_tail_input(be, params, rng):
    """A 127,008-value, 16-ciphertext packed vector shaped like conv1's
    squared output (fresh encryptions of small values)."""
    s = params.slot_count
    vals = rng.integers(0, 64, 8 * 126 * 126)
    chunks = [vals[i:i + s] for i in range(0, vals.size, s)]
    return I.PackedVector(vals.size, s, be.encrypt_many(chunks), shape=(8, 126, 126)), vals


def test_config3_tail_planned_equals_serial():
    """Config 3's conv2 (4 filters 3x3x8 over a 16-ciphertext input, 15,376
    rows) + square + FC: batched planner == per-row loop on limbs, levels,
    CostReport and decrypted logits."""
    from paper_1901_10074_b200.fv import FvBackend

    _, net = config_network(3)
    params = config_params(3)
    tail = I.NetworkSpec(net.layers[2:], (8, 126, 126))
    runs = []
    for planned in (True, False):
        be = FvBackend(params, rng=np.random.default_rng(1234))
        x, vals = _config3_tail_input(be, params, np.random.default_rng(33))
        out, trace = _run_network(be, tail, x, planned)
        logits = [int(v) for v in I.decrypt_logits(be, out)]
        runs.append((trace, be.cost_report().as_dict(), logits))
        del be, x, out
        _free()
    (tp, cp, lp), (ts, cs, ls) = runs
    assert tp == ts
    assert cp == cs
    assert lp == ls
    want = centred_mod(plaintext_forward(tail, vals.reshape(8, 126, 126)),
                       params.plain_modulus)
    assert lp == want


def test_config3_conv1_tile_planned_equals_serial():
    """A 2,048-row tile of config 3's conv1 (rows spanning the three channels
    and the first input-ciphertext boundary): planner == per-row loop."""
    from paper_1901_10074_b200.fv import FvBackend

    img, net = config_network(3)
    params = config_params(3)
    runs = []
    for planned in (True, False):
        be = FvBackend(params, rng=np.random.default_rng(1234))
        pv = I.pack_image(be, img)
        rows = I.compile_conv(net.layers[0], pv.slots_used)[:2048]
        out = (I.layer_eval(be, rows, pv) if planned
               else I._serial_layer_eval(be, rows, pv, True, 1))
        runs.append((_digests(out), [ct.level_used for ct in out.cts],
                     be.cost_report().as_dict()))
        del be, pv, out
        _free()
    assert runs[0] == runs[1]


def test_config5_encryption_stream_matches_reference():
    """Config 5: the first images of the 256-image stream, encrypted in
    sequence under one key (keygen and every encryption drawing from one
    Generator), equal the reference's ciphertexts; their logits are exact."""
    from paper_1901_10074_b200.fv import FvBackend

    g = _gold("config5_enc.json")
    imgs = batch_images(len(g["enc"]), seed=g["image_seed"])
    _, net = config_network(2)
    params = config_params(5)
    be = FvBackend(params, rng=np.random.default_rng(g["key_seed"]))
    for i, img in enumerate(imgs):
        pv = I.pack_image(be, img)
        assert _digests(pv) == g["enc"][i], f"image {i}"
        if i < 2:
            logits = [int(v) for v in I.decrypt_logits(be, I.infer(be, net, pv))]
            assert logits == centred_mod(plaintext_forward(net, img), params.plain_modulus)
