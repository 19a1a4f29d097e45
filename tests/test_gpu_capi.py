"""The object-level C-ABI (csrc/api.cu) against the CPU oracle.

SURVEY.md 8(b) lists the surface a host without torch needs: key upload in
the reference's stored form, ciphertext buffers with host upload/download,
encrypt/decrypt, add/add_plain/cmult, rotate(ct, g, key) and mult with
relinearisation.  Two drivers:

* ctypes, with the keys and ciphertexts of the ORACLE (the reference's
  algorithm, pinned by tests/test_oracle.py) in the reference's host layout:
  uploaded, operated on, downloaded, and compared limb for limb;
* tests/c_host/hefv_host.c, a plain-C program linked only against
  libhefv.so and the CUDA runtime, fed the same material through a file.

Both the per-prime (k = 4) and the aux-basis (k = 10) key switch are covered.
"""

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import fv_oracle as O
from paper_1901_10074_b200.params import BackendParams

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _pair(bits):
    from paper_1901_10074_b200.fv import FvBackend

    p = BackendParams(ring_dimension=1024, coeff_modulus_bits=bits, plain_modulus=12289,
                      slot_count=512, depth_budget=4)
    return (FvBackend(p, rng=np.random.default_rng(5)),
            O.OracleFvBackend(p, rng=np.random.default_rng(5)))


def _stack(lst):
    return np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.int64) for x in lst]))


@pytest.fixture(scope="module", params=[120, 300], ids=["k4_per_prime", "k10_aux"])
def pair(request):
    gpu, orc = _pair(request.param)
    assert gpu.ctx.ks_aux == (request.param == 300)
    return gpu, orc


def test_capi_ops_from_reference_keys(pair):
    import torch

    gpu, orc = pair
    ctx = gpu.ctx
    st = ctx.stream()
    k, n = ctx.k, ctx.n
    rng = np.random.default_rng(9)
    t = gpu.params.plain_modulus
    v = rng.integers(0, t, n // 2)
    w = rng.integers(0, t, n // 2)
    oa, ob = orc.encrypt(v), orc.encrypt(w)

    def key(sk):
        h = C.c_void_p()
        body, mask = _stack(sk.body), _stack(sk.mask)
        ctx.call("hefv_key_upload", body.ctypes.data, mask.ctypes.data, C.byref(h), st)
        return h

    def ct(parts):
        d = C.c_void_p()
        ctx.call("hefv_ct_alloc", 2, C.byref(d))
        host = _stack(parts)
        ctx.call("hefv_ct_upload", host.ctypes.data, 2, d, st)
        return d

    def down(d):
        host = np.empty((2, k, n), dtype=np.int64)
        ctx.call("hefv_ct_download", d, 2, host.ctypes.data, st)
        return host

    relin, rot1 = key(orc.keys.relin), key(orc.keys.galois[1])
    da, db = ct(oa.parts), ct(ob.parts)
    assert np.array_equal(down(da), _stack(oa.parts))
    out = C.c_void_p()
    ctx.call("hefv_ct_alloc", 2, C.byref(out))
    slots = torch.from_numpy(np.asarray(w, dtype=np.int64)).cuda()
    cases = [
        ("rotate", lambda: ctx.call("hefv_rotate", da, 3, rot1, out, st), orc.rotate(oa, 1)),
        ("mult", lambda: ctx.call("hefv_mult", da, db, relin, out, st), orc.mult(oa, ob)),
        ("square", lambda: ctx.call("hefv_mult", da, da, relin, out, st), orc.mult(oa, oa)),
        ("add", lambda: ctx.call("hefv_add", da, db, 2, out, st), orc.add(oa, ob)),
        ("add_plain", lambda: ctx.call("hefv_add_plain", da, 2, slots.data_ptr(), out, st),
         orc.add_plain(oa, w)),
        ("cmult", lambda: ctx.call("hefv_cmult", da, 2, slots.data_ptr(), out, st),
         orc.cmult(oa, w)),
    ]
    for name, run, want in cases:
        run()
        assert np.array_equal(down(out), _stack(want.parts)), name
    # in place: out may alias the input
    ctx.call("hefv_rotate", da, 3, rot1, da, st)
    assert np.array_equal(down(da), _stack(orc.rotate(oa, 1).parts))
    # encrypt / decrypt through the slot entry points (host-drawn randomness)
    pk = gpu._pk_mont
    u = np.asarray(ctx.rand_ternary(np.random.default_rng(3)), dtype=np.int8)[None]
    e1 = np.zeros_like(u)
    e2 = np.zeros_like(u)
    enc = torch.empty((1, 2, k, n), dtype=torch.int32, device="cuda")
    ud, e1d, e2d = (torch.from_numpy(x).cuda() for x in (u, e1, e2))
    ctx.call("hefv_encrypt_slots", pk.data_ptr(), ud.data_ptr(), e1d.data_ptr(), e2d.data_ptr(),
             slots.data_ptr(), enc.data_ptr(), 1, st)
    dec = torch.empty((1, n // 2), dtype=torch.int64, device="cuda")
    ctx.call("hefv_decrypt_slots", enc.data_ptr(), 2, gpu._s_mont.data_ptr(),
             gpu._s2_mont.data_ptr(), dec.data_ptr(), 1, st)
    assert np.array_equal(dec.cpu().numpy()[0], np.asarray(w) % t)
    for h in (relin, rot1):
        nat_free_key(h)
    for d in (da, db, out):
        ctx.call("hefv_ct_free", d)


def nat_free_key(h):
    from paper_1901_10074_b200 import _native as nat

    return nat.load().hefv_key_free(h)


def test_capi_rejects_bad_input(pair):
    from paper_1901_10074_b200.errors import NativeError

    gpu, orc = pair
    ctx = gpu.ctx
    st = ctx.stream()
    k, n = ctx.k, ctx.n
    d = C.c_void_p()
    ctx.call("hefv_ct_alloc", 2, C.byref(d))
    bad = np.zeros((2, k, n), dtype=np.int64)
    bad[1, k - 1, 7] = ctx.q_primes[k - 1]  # == p_j: outside [0, p_j)
    with pytest.raises(NativeError, match="outside"):
        ctx.call("hefv_ct_upload", bad.ctypes.data, 2, d, st)
    body = _stack(orc.keys.relin.body)
    mask = _stack(orc.keys.relin.mask).copy()
    mask[0, 0, 0] = -1
    h = C.c_void_p()
    with pytest.raises(NativeError, match="outside"):
        ctx.call("hefv_key_upload", body.ctypes.data, mask.ctypes.data, C.byref(h), st)
    with pytest.raises(NativeError, match="odd"):
        ctx.call("hefv_rotate", d, 4, gpu.keys.galois[1].handle, d, st)
    ctx.call("hefv_ct_free", d)


def test_c_host_program(pair, tmp_path):
    """tests/c_host/hefv_host.c: setup, key upload, ct upload, rotate / mult /
    add / add_plain / cmult, download -- no Python or torch on that side."""
    import __graft_entry__ as G

    exe = G._build_c_host()
    gpu, orc = pair
    rec = gpu.ctx.setup_record
    k, n = gpu.ctx.k, gpu.ctx.n
    rng = np.random.default_rng(11)
    t = gpu.params.plain_modulus
    v, w = rng.integers(0, t, n // 2), rng.integers(0, t, n // 2)
    oa, ob = orc.encrypt(v), orc.encrypt(w)
    src = tmp_path / "in.bin"
    with open(src, "wb") as f:
        np.array([rec["log_n"], len(rec["primes32"]), len(rec["primes64"]), rec["k"], rec["a"],
                  rec["t_index"], rec["wq"], rec["wm"], rec["ks_aux_base"]],
                 dtype=np.int64).tofile(f)
        for name in ("primes32", "psi32"):
            np.asarray(rec[name], dtype=np.uint32).tofile(f)
        for name in ("primes64", "psi64"):
            np.asarray(rec[name], dtype=np.uint64).tofile(f)
        np.asarray(rec["slot_to_ev"], dtype=np.int32).tofile(f)
        for name in ("q", "qhalf", "qhat", "qhat_inv", "m", "mhalf", "mhat", "mhat_inv",
                     "delta_mod"):
            np.asarray(rec[name], dtype=np.uint32).tofile(f)
        for sk in (orc.keys.relin, orc.keys.galois[1]):
            _stack(sk.body).tofile(f)
            _stack(sk.mask).tofile(f)
        _stack(oa.parts).tofile(f)
        _stack(ob.parts).tofile(f)
        np.asarray(w, dtype=np.uint64).tofile(f)
    dst = tmp_path / "out.bin"
    res = subprocess.run([str(exe), str(src), str(dst)], capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr
    got = np.fromfile(dst, dtype=np.int64).reshape(5, 2, k, n)
    wants = [orc.rotate(oa, 1), orc.mult(oa, ob), orc.add(oa, ob), orc.add_plain(oa, w),
             orc.cmult(oa, w)]
    for i, want in enumerate(wants):
        assert np.array_equal(got[i], _stack(want.parts)), ["rotate", "mult", "add", "add_plain",
                                                             "cmult"][i]


def test_layer_rows_rejects_bad_plans(pair):
    """hefv_layer_rows validates the host plan before any launch."""
    import torch

    from paper_1901_10074_b200.errors import NativeError

    gpu, _ = pair
    ctx = gpu.ctx
    st = ctx.stream()
    k, n = ctx.k, ctx.n
    x = torch.zeros((1, 2, k, n), dtype=torch.int32, device="cuda")
    out = torch.zeros((2, 2, k, n), dtype=torch.int32, device="cuda")
    galois = gpu.keys.galois
    offs = np.array(sorted(galois), dtype=np.int32)
    handles = (C.c_void_p * len(offs))(*[galois[int(o)].handle.value for o in offs])

    def call(row_out, plain_seg, n_iter=1, work_words=None, slot=0, key_offs=offs):
        R = len(row_out)
        row_out = np.asarray(row_out, dtype=np.int32)
        row_off = np.zeros(R, dtype=np.int32)
        row_ptr = np.arange(R + 1, dtype=np.int64)
        plain_seg = np.asarray(plain_seg, dtype=np.int32)
        plain_ptr = np.arange(R + 1, dtype=np.int64)
        slot_idx = np.full(R, slot, dtype=np.int32)
        slot_val = np.ones(R, dtype=np.uint64)
        words = C.c_int64()
        ctx.call("hefv_layer_rows_work_words", 1, R, row_ptr.ctypes.data, 4, C.byref(words))
        work = torch.empty(words.value, dtype=torch.int32, device="cuda")
        ww = words.value if work_words is None else work_words
        ws, cap = (None, 0)
        if ctx.ks_aux:
            from paper_1901_10074_b200.planner import _ks_workspace

            wst, cap = _ks_workspace(ctx, 4)
            ws = wst.data_ptr()
        ctx.call("hefv_layer_rows", x.data_ptr(), 1, R, row_out.ctypes.data, row_off.ctypes.data,
                 None, row_ptr.ctypes.data, plain_seg.ctypes.data, plain_ptr.ctypes.data,
                 slot_idx.ctypes.data, slot_val.ctypes.data, n_iter, gpu.params.slot_count,
                 len(key_offs), key_offs.ctypes.data, handles, out.data_ptr(), 2, 4,
                 work.data_ptr(), ww, ws, cap, st)

    call([0, 1], [0, 0])  # a valid two-row plan runs
    with pytest.raises(NativeError, match="grouped by output"):
        call([1, 0], [0, 0])
    with pytest.raises(NativeError, match="segment outside"):
        call([0, 1], [0, 3])
    with pytest.raises(NativeError, match="workspace too small"):
        call([0, 1], [0, 0], work_words=16)
    with pytest.raises(NativeError, match="outside \\[0, N/2\\)"):
        call([0, 1], [0, 0], slot=n)
    with pytest.raises(NativeError, match="power-of-two Galois key"):
        call([0, 1], [0, 0], n_iter=12, key_offs=offs[:1])
