"""The drop-in proof: the reference's OWN callers, unmodified, on the GPU backend.

The reference package is installed (git-ignored, test-only) in
``baseline/_ref`` by the recipe in DESIGN.md ("Reference install"); the
product never imports it.  These tests drive ``hepack.inference``
(``pack_image`` / ``infer`` / ``layer_eval`` / ``decrypt_logits``),
``hepack.fv.run_sequence`` / ``fv_conformance``, ``hepack.matrix`` and
``hepack.serialize`` with ``GpuFvBackend`` (paper_1901_10074_b200.dropin)
and compare with goldens the reference itself produced:

* unpatched: the reference's per-row ``layer_eval`` issues one GPU op per
  homomorphic operation;
* patched: ``layer_eval`` with the three-line dispatch of INTEGRATION.md
  (``dropin.layer_eval_hook``) runs the batched planner -- same limbs,
  levels, CostReport.
"""

import hashlib
import io
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle.fv_oracle import limb_digest
from paper_1901_10074_b200 import dropin
from paper_1901_10074_b200.configs import config_network
from paper_1901_10074_b200.params import profile

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
GOLD = ROOT / "tests" / "golden"


def _gold(name):
    return json.loads((GOLD / name).read_text())


@pytest.fixture(scope="module")
def hepack():
    if not (REF / "hepack" / "__init__.py").exists():
        pytest.skip("reference not installed in baseline/_ref (see DESIGN.md)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import hepack as H
    import hepack.fv
    import hepack.inference
    import hepack.matrix
    import hepack.serialize  # noqa: F401

    assert Path(H.__file__).resolve().is_relative_to(REF.resolve())
    return H


@pytest.fixture
def patched(hepack, monkeypatch):
    """The reference's layer_eval with the INTEGRATION.md dispatch (also the
    name hepack.matrix imported it under)."""
    hook = dropin.layer_eval_hook(hepack.inference.layer_eval)
    monkeypatch.setattr(hepack.inference, "layer_eval", hook)
    monkeypatch.setattr(hepack.matrix, "layer_eval", hook)
    return hook


# ---- CPU: the binding itself ---------------------------------------------------
def test_gpu_backend_class_is_both(hepack):
    from paper_1901_10074_b200.fv import FvBackend

    cls = dropin.gpu_backend_class(hepack.fv)
    assert issubclass(cls, FvBackend) and issubclass(cls, hepack.fv.FvBackend)
    assert cls is dropin.gpu_backend_class(hepack.fv)
    # every contract method resolves to the GPU implementation, not the reference's
    for name in ("encrypt", "decrypt", "add", "add_plain", "mult", "cmult", "rotate",
                 "all_sum", "partial_sum", "_encrypt", "_decrypt", "_add", "_add_plain",
                 "_mult", "_cmult", "_rotate", "decrypt_poly", "encode", "decode", "release",
                 "cost_report", "one_hot", "as_plain", "__init__"):
        owner = next(k for k in cls.__mro__ if name in vars(k))
        assert owner.__module__.startswith("paper_1901_10074_b200"), (name, owner)


def test_layer_eval_hook_dispatch(hepack):
    calls = []

    class Batched:
        def layer_eval_batched(self, rows, x, skip, scale):
            calls.append((rows, x, skip, scale))
            return "planned"

    def original(backend, rows, x, skip_zero_segments=True, threads=1, scale_factor=1):
        calls.append("serial")
        return "serial"

    hook = dropin.layer_eval_hook(original)
    assert hook(Batched(), [1], "x", True, 1, 4) == "planned"
    assert calls[-1] == ([1], "x", True, 4)
    assert hook(object(), [1], "x") == "serial"
    # the real reference function is left intact for every other backend
    sim = hepack.SimBackend(hepack.params.profile("desk"))
    x = hepack.inference.pack_image(sim, np.arange(16).reshape(1, 4, 4))
    rows = hepack.inference.compile_fc(
        hepack.inference.FcSpec(1, np.ones((1, 16), dtype=np.int64), np.zeros(1, np.int64)),
        x.slots_used)
    out = dropin.layer_eval_hook(hepack.inference.layer_eval)(sim, rows, x)
    assert int(sim.decrypt(out.cts[0])[0]) == sum(range(16))


# ---- GPU: the reference's callers on the GPU backend ------------------------------------
def _be(hepack, name, seed):
    return dropin.gpu_backend_class(hepack.fv)(profile(name), rng=np.random.default_rng(seed))


def _ref_net(hepack, cfg):
    """The reference's own NetworkSpec objects for a config (same draws as
    configs.config_network)."""
    img, net = config_network(cfg)
    R = hepack.inference
    layers = []
    for layer in net.layers:
        kind = type(layer).__name__
        if kind == "ConvSpec":
            layers.append(R.ConvSpec(layer.filters, layer.kernel, layer.stride, layer.in_shape,
                                     layer.weights, layer.biases))
        elif kind == "FcSpec":
            layers.append(R.FcSpec(layer.out_neurons, layer.weights, layer.biases))
        else:
            layers.append(R.SquareSpec())
    return img, R.NetworkSpec(layers, net.input_shape)


@pytest.mark.gpu
@pytest.mark.parametrize("with_hook", [False, True])
def test_reference_infer_config1(hepack, with_hook, request):
    """hepack.inference.pack_image -> infer -> decrypt_logits on the GPU
    backend: every layer's limbs, the logits and the CostReport equal the
    reference's own run (tests/golden/config1.json)."""
    if with_hook:
        request.getfixturevalue("patched")
    g = _gold("config1.json")
    R = hepack.inference
    img, net = _ref_net(hepack, 1)
    be = _be(hepack, "desk", g["key_seed"])
    pv = R.pack_image(be, img)
    assert [limb_digest(ct.parts) for ct in pv.cts] == g["enc"]
    out = R.infer(be, net, pv)
    assert type(out) is R.PackedVector
    assert [limb_digest(ct.parts) for ct in out.cts] == g["layers"][-1]
    assert [int(v) for v in R.decrypt_logits(be, out)] == g["logits"]
    assert be.cost_report().as_dict() == g["cost"]


@pytest.mark.gpu
def test_reference_run_sequence_and_conformance(hepack):
    """hepack.fv.run_sequence over make_golden.op_suite's operations: limbs,
    levels and CostReport equal the reference's (tests/golden/fv_desk.json);
    hepack.fv.fv_conformance against the reference's simulator holds."""
    g = _gold("fv_desk.json")
    ops_g = g["ops"]
    be = _be(hepack, "desk", g["seed"])
    rng = np.random.default_rng(g["data_seed"])
    slots, t = be.params.slot_count, be.params.plain_modulus
    v = rng.integers(0, t, slots)
    w = rng.integers(0, t, slots)
    ones = [1] * 100
    ops = [("enc", v), ("enc", w), ("add", 0, 1), ("add_plain", 0, w), ("cmult", 0, w),
           ("rotate", 0, 1), ("rotate", 0, 129), ("rotate", 0, -17), ("mult", 0, 1),
           ("mult", 0, 0), ("cmult", 0, ones), ("asum", 10, 100), ("psum", 0, 8)]
    stack = hepack.fv.run_sequence(be, ops)
    names = [None, None, "add", "add_plain", "cmult", "rotate1", "rotate129", "rotate-17",
             "mult", "square", None, "allsum", "psum8"]
    assert limb_digest(stack[0].parts) == ops_g["enc_a"]
    assert limb_digest(stack[1].parts) == ops_g["enc_b"]
    for ct, name in zip(stack, names):
        if name:
            assert limb_digest(ct.parts) == ops_g[name], name
            assert ct.level_used == ops_g[name + "_level"], name
    assert be.cost_report().as_dict() == ops_g["cost"]

    sim = hepack.SimBackend(hepack.params.profile("desk"))
    be2 = _be(hepack, "desk", 3)
    small = [("enc", v), ("enc", w), ("mult", 0, 1), ("rotate", 2, 5), ("cmult", 3, w),
             ("asum", 4, 64), ("psum", 0, 16), ("add_plain", 1, v)]
    assert hepack.fv.fv_conformance(be2, sim, small)


@pytest.mark.gpu
@pytest.mark.parametrize("with_hook", [False, True])
def test_reference_matrix_suite(hepack, with_hook, request):
    """hepack.matrix (packings, conversion, transpose, mat_mul on one and on
    several ciphertexts, plain_mat_mul through layer_eval) on the GPU backend
    equals the reference's own run (tests/golden/matrix.json)."""
    from goldens import matrix_suite

    if with_hook:
        request.getfixturevalue("patched")
    g = _gold("matrix.json")
    be = _be(hepack, "desk", g["key_seed"])
    got = matrix_suite(be, hepack.matrix, np.random.default_rng(g["data_seed"]))
    for key in ("mm3", "mm3_plain", "mm5s13", "mm5s13_plain", "conv_cp", "transpose_keep", "pmm",
                "pmm_plain", "cost"):
        assert got[key] == g[key], key


@pytest.mark.gpu
def test_reference_serialize(hepack, tmp_path):
    """hepack.serialize on the GPU backend: records byte-identical to the
    files the reference wrote (tests/golden/serialize.json); FV records read
    back through the reference's reader (which requires an FvBackend
    instance) and computed on directly; a reference key directory loads into
    the GPU backend."""
    S = hepack.serialize
    g = _gold("serialize.json")
    p = profile("desk")
    be = _be(hepack, "desk", g["key_seed"])
    rng = np.random.default_rng(g["data_seed"])
    v = rng.integers(0, p.plain_modulus, p.slot_count)
    ct = be.encrypt(v)
    buf = io.BytesIO()
    S.write_ciphertext(buf, ct, p)
    assert hashlib.sha256(buf.getvalue()).hexdigest() == g["ct_record"]
    buf.seek(0)
    back = S.read_ciphertext(buf, be)
    assert type(back) is hepack.fv.FvCiphertext            # the reference's host record
    assert np.array_equal(be.decrypt(back), v)
    assert limb_digest(be.add(back, ct).parts) == limb_digest(be.add(ct, ct).parts)
    img, _ = config_network(1)
    pv = hepack.inference.pack_image(be, img)
    S.write_encrypted_image(tmp_path / "img.enc", pv, p)
    assert hashlib.sha256((tmp_path / "img.enc").read_bytes()).hexdigest() == g["image"]
    again = S.read_encrypted_image(tmp_path / "img.enc", be)
    assert [limb_digest(c.parts) for c in again.cts] == [limb_digest(c.parts) for c in pv.cts]
    S.write_logits(tmp_path / "logits.bin", [ct, pv.cts[0]], [(0, 0), (0, 1)], p)
    assert hashlib.sha256((tmp_path / "logits.bin").read_bytes()).hexdigest() == g["logits"]
    fp = hepack.fv.FvParams(n=be.ctx.n, t=be.ctx.t, q_primes=be.ctx.q_primes)
    S.write_keyset(tmp_path / "keys", be.keys, fp, p)
    for name, digest in g["keyset"].items():
        assert hashlib.sha256((tmp_path / "keys" / name).read_bytes()).hexdigest() == digest, name
    # the reference's reader + the GPU backend constructed on its KeySet
    ks = S.read_keyset(tmp_path / "keys")
    be2 = dropin.gpu_backend_class(hepack.fv)(p, keys=ks, rng=np.random.default_rng(1))
    assert np.array_equal(be2.decrypt(back), v)
    assert np.array_equal(be2.decrypt(be2.rotate(back, 3)), np.roll(v, -3))
    # a corrupt record fails on the host before anything reaches the device
    bad = bytearray(buf.getvalue())
    bad[-8:] = (1 << 62).to_bytes(8, "little")
    rec = S.read_ciphertext(io.BytesIO(bytes(bad)), be)
    from paper_1901_10074_b200.errors import FormatError

    with pytest.raises(FormatError):
        be.decrypt(rec)
