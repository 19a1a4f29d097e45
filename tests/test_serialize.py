"""Wire formats (serialize.py of the reference, /root/reference/pkg/src/hepack/
serialize.py): byte-identical records, round trips and error behaviour.

CPU tests pin the byte layout with the oracle's ciphertexts and keys against
the digests of files the reference itself wrote (tests/golden/serialize.json)
and cover the simulator records; the GPU tests write the same files from
device-resident ciphertexts/keys and load key directories straight into the
device layout."""

import hashlib
import io
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import config_network
from paper_1901_10074_b200.engine import SimBackend
from paper_1901_10074_b200.errors import FormatError
from paper_1901_10074_b200.params import profile
from paper_1901_10074_b200.serialize import (
    read_ciphertext,
    read_encrypted_image,
    read_logits,
    write_ciphertext,
    write_encrypted_image,
    write_keyset,
    write_logits,
)

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "serialize.json").read_text())
KEYFILES = ("params.json", "secret.bin", "public.bin", "relin.bin", "galois.bin")


def _sha(data: bytes) -> str:
    return hashlib.sha256(data).hexdigest()


@pytest.fixture
def desk():
    return SimBackend(profile("desk"))


def _write_all(tmp_path, be, params, keys, fp):
    """The files make_golden.gen_serialize writes, from backend ``be``."""
    rng = np.random.default_rng(GOLD["data_seed"])
    v = rng.integers(0, params.plain_modulus, params.slot_count)
    ct = be.encrypt(v)
    buf = io.BytesIO()
    write_ciphertext(buf, ct, params)
    img, _ = config_network(1)
    pv = I.pack_image(be, img)
    write_encrypted_image(tmp_path / "img.enc", pv, params)
    write_logits(tmp_path / "logits.bin", [ct, pv.cts[0]], [(0, 0), (0, 1)], params)
    write_keyset(tmp_path / "keys", keys, fp, params)
    return v, ct, pv, buf.getvalue()


def _check_bytes(tmp_path, record):
    assert len(record) == GOLD["ct_record_len"]
    assert _sha(record) == GOLD["ct_record"]
    assert _sha((tmp_path / "img.enc").read_bytes()) == GOLD["image"]
    assert _sha((tmp_path / "logits.bin").read_bytes()) == GOLD["logits"]
    for name in KEYFILES:
        assert _sha((tmp_path / "keys" / name).read_bytes()) == GOLD["keyset"][name], name


@pytest.mark.slow
def test_oracle_records_byte_identical_to_reference(tmp_path):
    """Byte layout pin on CPU: oracle ciphertexts/keys (limb-identical to the
    reference's) written by this module hash to the reference's own files."""
    from oracle.fv_oracle import OracleFvBackend, OracleParams

    params = profile("desk")
    be = OracleFvBackend(params, rng=np.random.default_rng(GOLD["key_seed"]))
    _, _, _, record = _write_all(tmp_path, be, params, be.keys, OracleParams.from_backend(params))
    _check_bytes(tmp_path, record)


def test_sim_ciphertext_roundtrip(desk, rng):
    v = rng.integers(0, desk.params.plain_modulus, desk.params.slot_count)
    ct = desk.encrypt(v)
    buf = io.BytesIO()
    write_ciphertext(buf, ct, desk.params)
    buf.seek(0)
    again = read_ciphertext(buf, desk)
    assert again.level_used == ct.level_used
    assert np.array_equal(desk.decrypt(again), desk.decrypt(ct))


def test_ciphertext_rejects_wrong_params(desk):
    buf = io.BytesIO()
    write_ciphertext(buf, desk.encrypt([1, 2, 3]), desk.params)
    buf.seek(0)
    with pytest.raises(FormatError):
        read_ciphertext(buf, SimBackend(desk.params.replace(plain_modulus=40961)))


def test_bad_magic_and_kind(desk):
    with pytest.raises(FormatError):
        read_ciphertext(io.BytesIO(b"XXXX" + bytes(20)), desk)
    buf = io.BytesIO()
    write_ciphertext(buf, desk.encrypt([1]), desk.params)
    raw = bytearray(buf.getvalue())
    raw[4] = 9
    with pytest.raises(FormatError):
        read_ciphertext(io.BytesIO(bytes(raw)), desk)
    raw[4], raw[5] = 1, 7  # version
    with pytest.raises(FormatError):
        read_ciphertext(io.BytesIO(bytes(raw)), desk)


def test_encrypted_image_roundtrip(tmp_path, desk, rng):
    img = rng.integers(0, 4, (1, 6, 5))
    pv = I.pack_image(desk, img, slots_used=7)
    path = tmp_path / "img.enc"
    write_encrypted_image(path, pv, desk.params)
    again = read_encrypted_image(path, desk)
    assert again.shape == (1, 6, 5) and again.slots_used == 7
    for p, v in enumerate(img.reshape(-1)):
        assert desk.decrypt(again.cts[p // 7])[p % 7] == v


def test_logits_roundtrip(tmp_path, desk, rng):
    pv = I.pack_image(desk, rng.integers(0, 9, (1, 1, 10)))
    slot_map = [(i // pv.slots_used, i % pv.slots_used) for i in range(10)]
    path = tmp_path / "logits.bin"
    write_logits(path, pv.cts, slot_map, desk.params)
    cts, again_map = read_logits(path, desk)
    assert again_map == slot_map
    assert len(cts) == len(pv.cts)
    assert np.array_equal(desk.decrypt(cts[0]), desk.decrypt(pv.cts[0]))


def test_truncated_file_raises(tmp_path, desk):
    pv = I.pack_image(desk, np.ones((1, 2, 2), dtype=int))
    path = tmp_path / "img.enc"
    write_encrypted_image(path, pv, desk.params)
    data = path.read_bytes()
    path.write_bytes(data[: len(data) // 2])
    with pytest.raises(FormatError):
        read_encrypted_image(path, desk)


def test_sim_backend_rejects_fv_record(desk):
    """An FV record (host-part ciphertext; no device needed to write it) is
    refused by the simulator backend (serialize.py:108-110)."""
    from paper_1901_10074_b200.fv import FvCiphertext

    params = desk.params
    ct = FvCiphertext([np.zeros((6, 4096), np.int64)] * 2, 0, params)
    buf = io.BytesIO()
    write_ciphertext(buf, ct, params)
    buf.seek(0)
    with pytest.raises(FormatError):
        read_ciphertext(buf, desk)


def test_missing_key_directory(tmp_path):
    from paper_1901_10074_b200.serialize import read_keyset

    with pytest.raises(FormatError):
        read_keyset(tmp_path / "nope")


# ---- GPU -------------------------------------------------------------------------


@pytest.mark.gpu
def test_gpu_records_byte_identical_to_reference(tmp_path):
    """Device ciphertexts and keys written to the reference's wire format hash
    to the files the reference wrote for the same seeds."""
    from paper_1901_10074_b200.fv import FvBackend, FvParams

    params = profile("desk")
    be = FvBackend(params, rng=np.random.default_rng(GOLD["key_seed"]))
    _, _, _, record = _write_all(tmp_path, be, params, be.keys, FvParams.from_backend(params))
    _check_bytes(tmp_path, record)


@pytest.mark.gpu
def test_gpu_keyset_and_ciphertext_roundtrip(tmp_path):
    """Key directory -> device KeySet (no keygen): old ciphertexts decrypt,
    and rotations/squares under the loaded keys are limb-identical to the
    ones under the original device keys."""
    from oracle.fv_oracle import limb_digest
    from paper_1901_10074_b200.fv import FvBackend, FvParams
    from paper_1901_10074_b200.serialize import read_keyset

    params = profile("desk")
    t = params.plain_modulus
    be = FvBackend(params, rng=np.random.default_rng(3))
    v = np.random.default_rng(8).integers(0, t, params.slot_count)
    ct = be.encrypt(v)
    buf = io.BytesIO()
    write_ciphertext(buf, ct, params)
    buf.seek(0)
    again = read_ciphertext(buf, be)
    assert limb_digest(again.parts) == limb_digest(ct.parts)
    assert np.array_equal(be.decrypt(again), v % t)

    write_keyset(tmp_path / "keys", be.keys, FvParams.from_backend(params), params)
    loaded = read_keyset(tmp_path / "keys")
    be2 = FvBackend(params, keys=loaded, rng=np.random.default_rng(11))
    assert np.array_equal(be2.decrypt(again), v % t)
    for off in (1, 5, 2047):
        assert limb_digest(be2.rotate(again, off).parts) == limb_digest(be.rotate(ct, off).parts)
    assert limb_digest(be2.mult(again, again).parts) == limb_digest(be.mult(ct, ct).parts)
    rot = be2.rotate(be2.encrypt(v), 5)
    assert np.array_equal(be2.decrypt(rot), np.roll(v % t, -5))
    # the loaded set writes back to identical files
    write_keyset(tmp_path / "keys2", loaded, FvParams.from_backend(params), params)
    for name in KEYFILES:
        assert (tmp_path / "keys" / name).read_bytes() == (tmp_path / "keys2" / name).read_bytes()


@pytest.mark.gpu
def test_gpu_keyset_rejects_other_params(tmp_path):
    from paper_1901_10074_b200.errors import ParamMismatchError
    from paper_1901_10074_b200.fv import FvBackend, FvParams
    from paper_1901_10074_b200.serialize import read_keyset

    params = profile("desk")
    be = FvBackend(params, rng=np.random.default_rng(3))
    write_keyset(tmp_path / "keys", be.keys, FvParams.from_backend(params), params)
    loaded = read_keyset(tmp_path / "keys")
    with pytest.raises(ParamMismatchError):
        FvBackend(params.replace(plain_modulus=40961), keys=loaded)

