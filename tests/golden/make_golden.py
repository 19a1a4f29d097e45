"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--retina]

Writes tests/golden/{ntt,primes,fv_desk,fv_tiny,config1}.json (and
retina.json with --retina, ~4 min).  Fixtures hold seeds, small inputs and
sha256 digests of the reference's int64 limbs (oracle.fv_oracle.limb_digest
layout), plus full vectors where they are small.  The reference is imported
only here; tests read the JSON.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent

from hepack import engine as R_engine  # noqa: E402
from hepack import fv as R_fv  # noqa: E402
from hepack import inference as R_inf  # noqa: E402
from hepack import ntt as R_ntt  # noqa: E402
from hepack.params import BackendParams, profile  # noqa: E402


def digest(parts) -> str:
    h = hashlib.sha256()
    for p in parts:
        h.update(np.ascontiguousarray(np.asarray(p, dtype=np.int64)).astype("<i8").tobytes())
    return h.hexdigest()


def vec_digest(v) -> str:
    return digest([np.asarray([int(x) for x in v], dtype=np.int64)])


def key_digest(sk) -> str:
    return digest(list(sk.body) + list(sk.mask))


def dump(name, obj):
    (HERE / name).write_text(json.dumps(obj, indent=1, sort_keys=True))
    print("wrote", name)


def gen_ntt():
    cases = []
    for n, bits in [(8, 30), (64, 30), (256, 30), (16, 20), (4096, 30), (16384, 30),
                    (32768, 30), (4096, 50), (16384, 60), (32768, 55), (65536, 60)]:
        p = R_ntt.find_ntt_primes(1, bits, 2 * n)[0]
        tr = R_ntt.NttPrime(p, n)
        rng = np.random.default_rng(n * 1000 + bits)
        a = np.array([int(rng.integers(0, p)) for _ in range(n)], dtype=object)
        fa = tr.fwd(a)
        case = {"n": n, "bits": bits, "p": p, "psi": tr.psi, "seed": n * 1000 + bits,
                "in_digest": vec_digest(a), "fwd_digest": vec_digest(fa),
                "fwd_head": [int(x) for x in fa[:4]],
                "inv_roundtrip": bool(all(int(x) == int(y) for x, y in zip(tr.inv(fa), a)))}
        if n <= 256:
            case["in"] = [int(x) for x in a]
            case["fwd"] = [int(x) for x in fa]
        cases.append(case)
    dump("ntt.json", {"cases": cases})


def gen_primes():
    out = {}
    for name in ("desk", "mnist", "retina"):
        fp = R_fv.FvParams.from_backend(profile(name))
        ctx = R_fv._FvContext(fp)
        out[name] = {"q": fp.q_primes, "aux": ctx.aux_primes, "t_psi": ctx.t_ntt.psi,
                     "q_psi": [tr.psi for tr in ctx.q_ntt],
                     "slot_to_ev_digest": vec_digest(ctx.slot_to_ev),
                     "gadget_digest": vec_digest([g % (1 << 61) for g in ctx.gadget])}
    p720 = profile("retina").replace(coeff_modulus_bits=720)
    fp = R_fv.FvParams.from_backend(p720)
    ctx = R_fv._FvContext(fp)
    out["retina-720"] = {"q": fp.q_primes, "aux": ctx.aux_primes}
    dump("primes.json", out)


def op_suite(be, rng, slots, t):
    """The op sequence replayed by the GPU/oracle tests (same order of draws)."""
    v = rng.integers(0, t, slots)
    w = rng.integers(0, t, slots)
    a = be.encrypt(v)
    b = be.encrypt(w)
    res = {"v": vec_digest(v), "w": vec_digest(w), "enc_a": digest(a.parts),
           "enc_b": digest(b.parts)}
    ops = [
        ("add", lambda: be.add(a, b)),
        ("add_plain", lambda: be.add_plain(a, w)),
        ("cmult", lambda: be.cmult(a, w)),
        ("rotate1", lambda: be.rotate(a, 1)),
        ("rotate129", lambda: be.rotate(a, 129 % slots)),
        ("rotate-17", lambda: be.rotate(a, -17)),
        ("mult", lambda: be.mult(a, b)),
        ("square", lambda: be.mult(a, a)),
        ("allsum", lambda: be.all_sum(be.cmult(a, [1] * min(100, slots)), min(100, slots))),
        ("psum8", lambda: be.partial_sum(a, 8)),
    ]
    for name, fn in ops:
        ct = fn()
        res[name] = digest(ct.parts)
        res[name + "_dec"] = vec_digest(be.decrypt(ct))
        res[name + "_level"] = ct.level_used
    res["decpoly_a"] = vec_digest(be.decrypt_poly(a))
    res["cost"] = be.cost_report().as_dict()
    return res


def gen_fv_desk():
    p = profile("desk")
    be = R_fv.FvBackend(p, rng=np.random.default_rng(77))
    k = be.keys
    out = {"seed": 77, "data_seed": 5,
           "secret": digest([k.secret]), "pk": digest(list(k.public)),
           "relin": key_digest(k.relin),
           "galois": {str(off): key_digest(sk) for off, sk in k.galois.items()}}
    out["ops"] = op_suite(be, np.random.default_rng(5), p.slot_count, p.plain_modulus)
    dump("fv_desk.json", out)


def gen_fv_tiny():
    p = BackendParams(ring_dimension=64, coeff_modulus_bits=120, plain_modulus=257, slot_count=32,
                      depth_budget=4)
    be = R_fv.FvBackend(p, rng=np.random.default_rng(5))
    rng = np.random.default_rng(9)
    v = rng.integers(0, 257, 32)
    a = be.encrypt(v)
    out = {"params": {"ring_dimension": 64, "coeff_modulus_bits": 120, "plain_modulus": 257,
                      "slot_count": 32, "depth_budget": 4},
           "key_seed": 5, "data_seed": 9,
           "enc": [p_.tolist() for p_ in a.parts],
           "square": [p_.tolist() for p_ in be.mult(a, a).parts],
           "rotate7": [p_.tolist() for p_ in be.rotate(a, 7).parts],
           "cmult": [p_.tolist() for p_ in be.cmult(a, v).parts]}
    dump("fv_tiny.json", out)


def net_for(cfg):
    rng = np.random.default_rng(cfg)
    if cfg == 1:
        img = rng.integers(0, 256, (1, 16, 16), dtype=np.int64)
        conv = R_inf.ConvSpec(2, (3, 3), (2, 2), (1, 16, 16), rng.integers(-4, 5, (2, 1, 3, 3)),
                              np.zeros(2, np.int64))
        fc = R_inf.FcSpec(2, rng.integers(-4, 5, (2, conv.out_len)), np.zeros(2, np.int64))
        return img, R_inf.NetworkSpec([conv, R_inf.SquareSpec(), fc], (1, 16, 16))
    img = rng.integers(0, 256, (1, 96, 96), dtype=np.int64)
    conv = R_inf.ConvSpec(5, (5, 5), (2, 2), (1, 96, 96), rng.integers(-8, 9, (5, 1, 5, 5)),
                          np.zeros(5, np.int64))
    fc = R_inf.FcSpec(2, rng.integers(-8, 9, (2, conv.out_len)), np.zeros(2, np.int64))
    return img, R_inf.NetworkSpec([conv, R_inf.SquareSpec(), fc], (1, 96, 96))


def gen_config1():
    img, net = net_for(1)
    be = R_fv.FvBackend(profile("desk"), rng=np.random.default_rng(1234))
    t0 = time.time()
    pv = R_inf.pack_image(be, img)
    enc = [digest(ct.parts) for ct in pv.cts]
    layers = []
    cur = pv
    for layer in net.layers:
        if isinstance(layer, R_inf.SquareSpec):
            nxt = R_inf.square_activation(be, cur)
        else:
            rows = (R_inf.compile_conv(layer, cur.slots_used) if isinstance(layer, R_inf.ConvSpec)
                    else R_inf.compile_fc(layer, cur.slots_used))
            nxt = R_inf.layer_eval(be, rows, cur)
        if cur is not pv:
            be.release(*cur.cts)
        cur = nxt
        layers.append([digest(ct.parts) for ct in cur.cts])
    logits = R_inf.decrypt_logits(be, cur)
    out = {"key_seed": 1234, "data_seed": 1, "enc": enc, "layers": layers,
           "logits": [int(x) for x in logits], "cost": be.cost_report().as_dict(),
           "seconds": time.time() - t0}
    dump("config1.json", out)


def gen_retina():
    p = profile("retina")
    t0 = time.time()
    be = R_fv.FvBackend(p, rng=np.random.default_rng(1234))
    tk = time.time() - t0
    img, net = net_for(2)
    k = be.keys
    pv = R_inf.pack_image(be, img)
    out = {"key_seed": 1234, "keygen_seconds": tk, "relin": key_digest(k.relin),
           "galois1": key_digest(k.galois[1]), "galois4096": key_digest(k.galois[4096]),
           "pk": digest(list(k.public)), "enc": [digest(ct.parts) for ct in pv.cts]}
    a = pv.cts[0]
    out["rotate1"] = digest(be.rotate(a, 1).parts)
    sq = be.mult(a, a)
    out["square"] = digest(sq.parts)
    out["square_dec_ok"] = bool(np.array_equal(
        np.asarray(be.decrypt(sq), dtype=object),
        np.asarray(be.decrypt(a), dtype=object) ** 2 % p.plain_modulus))
    # a subset of config-2 conv rows (all in output ciphertext 0)
    rows = R_inf.compile_conv(net.layers[0], pv.slots_used)
    pick = [0, 1, 47, 2500, 8191]
    t1 = time.time()
    res = R_inf.layer_eval(be, [rows[i] for i in pick], pv)
    out["rows_pick"] = pick
    out["rows_out"] = [digest(ct.parts) for ct in res.cts]
    out["rows_cost"] = be.cost_report().as_dict()
    out["rows_seconds"] = time.time() - t1
    dump("retina.json", out)


if __name__ == "__main__" and len(sys.argv) == 1 or "--retina" in sys.argv:
    gen_ntt()
    gen_primes()
    gen_fv_tiny()
    gen_fv_desk()
    gen_config1()
    if "--retina" in sys.argv:
        gen_retina()
    del R_engine


def gen_config3_rows():
    """Config 3 (retina with 24 q primes): keys, the 24 input encryptions and
    a subset of conv1 rows (all in output ciphertext 0) -- reference run."""
    p = profile("retina").replace(coeff_modulus_bits=720)
    t0 = time.time()
    be = R_fv.FvBackend(p, rng=np.random.default_rng(1234))
    tk = time.time() - t0
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (3, 256, 256), dtype=np.int64)
    c1 = R_inf.ConvSpec(8, (5, 5), (2, 2), (3, 256, 256), rng.integers(-8, 9, (8, 3, 5, 5)),
                        np.zeros(8, np.int64))
    pv = R_inf.pack_image(be, img)
    rows = R_inf.compile_conv(c1, pv.slots_used)
    pick = [0, 1, 126, 4095]
    t1 = time.time()
    res = R_inf.layer_eval(be, [rows[i] for i in pick], pv)
    out = {"key_seed": 1234, "data_seed": 3, "coeff_modulus_bits": 720,
           "relin": key_digest(be.keys.relin), "enc": [digest(ct.parts) for ct in pv.cts],
           "rows_pick": pick, "rows_out": [digest(ct.parts) for ct in res.cts],
           "rows_cost": be.cost_report().as_dict(), "keygen_seconds": tk,
           "rows_seconds": time.time() - t1}
    dump("config3_rows.json", out)


if __name__ == "__main__" and "--config3" in sys.argv:
    gen_config3_rows()


def gen_serialize():
    """Wire-format bytes written by the reference's own serialize module:
    sha256 of a FV ciphertext record, an encrypted image (config 1 input), a
    logits record, and each file of a desk key directory."""
    import io
    import tempfile

    from hepack import serialize as R_ser

    p = profile("desk")
    be = R_fv.FvBackend(p, rng=np.random.default_rng(77))
    rng = np.random.default_rng(5)
    v = rng.integers(0, p.plain_modulus, p.slot_count)
    ct = be.encrypt(v)
    buf = io.BytesIO()
    R_ser.write_ciphertext(buf, ct, p)
    out = {"key_seed": 77, "data_seed": 5,
           "ct_record": hashlib.sha256(buf.getvalue()).hexdigest(),
           "ct_record_len": len(buf.getvalue())}
    img, _ = net_for(1)
    pv = R_inf.pack_image(be, img)
    with tempfile.TemporaryDirectory() as d:
        R_ser.write_encrypted_image(f"{d}/img.enc", pv, p)
        out["image"] = hashlib.sha256(open(f"{d}/img.enc", "rb").read()).hexdigest()
        slot_map = [(0, 0), (0, 1)]
        R_ser.write_logits(f"{d}/logits.bin", [ct, pv.cts[0]], slot_map, p)
        out["logits"] = hashlib.sha256(open(f"{d}/logits.bin", "rb").read()).hexdigest()
        fp = R_fv.FvParams.from_backend(p)
        R_ser.write_keyset(f"{d}/keys", be.keys, fp, p)
        out["keyset"] = {name: hashlib.sha256(open(f"{d}/keys/{name}", "rb").read()).hexdigest()
                         for name in ("params.json", "secret.bin", "public.bin", "relin.bin",
                                      "galois.bin")}
    dump("serialize.json", out)


if __name__ == "__main__" and "--serialize" in sys.argv:
    gen_serialize()


def interleaved_net(inf):
    """Small interleaved-baseline net: conv with a bias, square, FC with an
    all-zero row (bias-only -> encryption) and a negative bias."""
    rng = np.random.default_rng(11)
    img = rng.integers(0, 16, (1, 6, 6), dtype=np.int64)
    conv = inf.ConvSpec(2, (3, 3), (2, 2), (1, 6, 6), rng.integers(-4, 5, (2, 1, 3, 3)),
                        np.array([3, 0], dtype=np.int64))
    w = rng.integers(-4, 5, (3, conv.out_len))
    w[2] = 0
    fc = inf.FcSpec(3, w, np.array([1, -2, 5], dtype=np.int64))
    return img, inf.NetworkSpec([conv, inf.SquareSpec(), fc], (1, 6, 6))


def gen_interleaved():
    img, net = interleaved_net(R_inf)
    be = R_fv.FvBackend(profile("desk"), rng=np.random.default_rng(1234))
    px = R_inf.pack_image_interleaved(be, img)
    enc = [digest(ct.parts) for ct in px]
    out = R_inf.interleaved_infer(be, net, px)
    logits = R_inf.decrypt_logits(be, out)
    dump("interleaved.json", {"key_seed": 1234, "enc": enc, "out": [digest(ct.parts) for ct in out],
                              "levels": [ct.level_used for ct in out],
                              "logits": [int(x) for x in logits],
                              "cost": be.cost_report().as_dict()})


if __name__ == "__main__" and "--interleaved" in sys.argv:
    gen_interleaved()


def gen_matrix():
    from hepack import matrix as R_mx

    sys.path.insert(0, str(HERE.parent.parent))
    sys.path.insert(0, str(HERE.parent))
    from goldens import matrix_suite

    be = R_fv.FvBackend(profile("desk"), rng=np.random.default_rng(1234))
    t0 = time.time()
    out = matrix_suite(be, R_mx, np.random.default_rng(17))
    out.update({"key_seed": 1234, "data_seed": 17, "seconds": time.time() - t0})
    dump("matrix.json", out)


if __name__ == "__main__" and "--matrix" in sys.argv:
    gen_matrix()


# ---- sharded reference: whole-layer limb goldens at retina ----------------
#
# The reference evaluates a layer one row at a time (inference.py:261-349);
# every row's piece is added into its output ciphertext, and limb-wise
# addition mod p_j is exact and commutative.  So a layer restricted to a row
# subset R (the other rows replaced by all-zero rows, which layer_eval skips
# without any operation, inference.py:303-309) splits into shards R_1..R_W
# whose outputs sum limb-wise to the output over R -- provided every shard
# places at least one row in every output ciphertext (otherwise layer_eval
# encrypts a fresh zero there, inference.py:339-341).  Each worker runs the
# unmodified reference (own keygen from default_rng(1234), so identical keys
# and input encryptions) on its shard; the parent sums the pieces mod p_j,
# then runs the reference's own square (and, for config 2, the FC layer) on
# the summed ciphertexts.  Digests of all of it go to rows_shard_c{2,3}.json.

SHARD_WORKERS = 8


def _popcount(x):
    return bin(x).count("1")


def rows_shard_picks(cfg):
    """Deterministic row picks (out_index values) and their shard split.

    Config 2 (10,580 conv rows, 2 output cts): every placement-hop count
    1..13 (rotation by -off = 8192-off, popcount hops, fv.py:422-425) in both
    output ciphertexts where it exists, off = 0, the rows whose 5x5 window
    straddles the input-ciphertext boundary (image rows 85/86 -> oy 41, 42)
    for every filter, first / last rows, and seeded random rows -> 64.
    Config 3 (rows list truncated to the first 16,384 conv1 rows = filter 0
    and the start of filter 1, 2 output cts): every row spans 3 channels
    (3-6 input segments); picks cover the input-ct boundary rows (input ct =
    32 image rows: oy 14, 15, 16 and 30, 31), placement hop counts, and the
    filter-0/1 boundary -> 32."""
    s = 8192
    if cfg == 2:
        total, f_len, ow, want = 10580, 2116, 46, 64
        picks = {0, s, total - 1, 1}
        for b in range(1, 14):
            for ct in (0, 1):
                lim = s if ct == 0 else total - s
                cands = [off for off in range(1, lim) if _popcount(s - off) == b]
                if cands:
                    picks.add(ct * s + cands[len(cands) // 2])
        for f in range(5):
            for oy in (41, 42):
                picks.add(f * f_len + oy * ow + 7 * f)
    else:
        total, f_len, ow, want = 16384, 15876, 126, 32
        picks = {0, s, total - 1, 8191, f_len - 1, f_len}
        for oy in (14, 15, 16, 30, 31, 62, 64):
            picks.add(oy * ow + (oy * 3) % ow)
        for b in (1, 4, 8, 11, 13):
            cands = [off for off in range(1, total - s) if _popcount(s - off) == b]
            if cands:
                picks.add(s + cands[len(cands) // 3])
    rng = np.random.default_rng(20 + cfg)
    while len(picks) < want:
        picks.add(int(rng.integers(0, total)))
    picks = sorted(picks)[:want] if len(picks) > want else sorted(picks)
    ct0 = [r for r in picks if r < s]
    ct1 = [r for r in picks if r >= s]
    assert len(ct1) >= SHARD_WORKERS and len(ct0) >= SHARD_WORKERS, (len(ct0), len(ct1))
    shards = [[] for _ in range(SHARD_WORKERS)]
    for i, r in enumerate(ct0):
        shards[i % SHARD_WORKERS].append(r)
    for i, r in enumerate(ct1):
        shards[i % SHARD_WORKERS].append(r)
    return total, picks, [sorted(sh) for sh in shards]


def _shard_setup(cfg):
    if cfg == 2:
        p = profile("retina")
        img, net = net_for(2)
        conv = net.layers[0]
    else:
        p = profile("retina").replace(coeff_modulus_bits=720)
        rng = np.random.default_rng(3)
        img = rng.integers(0, 256, (3, 256, 256), dtype=np.int64)
        conv = R_inf.ConvSpec(8, (5, 5), (2, 2), (3, 256, 256), rng.integers(-8, 9, (8, 3, 5, 5)),
                              np.zeros(8, np.int64))
        net = None
    return p, img, net, conv


def _masked_rows(rows, keep, total):
    out = []
    keep = set(keep)
    for i in range(total):
        r = rows[i]
        if i in keep:
            out.append(r)
        else:
            out.append(R_inf.WeightRow(out_index=r.out_index, length=r.length,
                                       slots_used=r.slots_used,
                                       positions=np.zeros(0, np.int64),
                                       values=np.zeros(0, np.int64), bias=0))
    return out


def _shard_worker(args):
    cfg, shard = args
    p, img, net, conv = _shard_setup(cfg)
    t0 = time.time()
    be = R_fv.FvBackend(p, rng=np.random.default_rng(1234))
    pv = R_inf.pack_image(be, img)
    total, _, _ = rows_shard_picks(cfg)
    rows = R_inf.compile_conv(conv, pv.slots_used)
    res = R_inf.layer_eval(be, _masked_rows(rows, shard, total), pv)
    return {"parts": [[np.asarray(x, dtype=np.int64) for x in ct.parts] for ct in res.cts],
            "levels": [ct.level_used for ct in res.cts],
            "cost": be.cost_report().as_dict(), "seconds": time.time() - t0,
            "enc": [digest(ct.parts) for ct in pv.cts]}


def gen_rows_shard(cfg):
    import multiprocessing as mp

    total, picks, shards = rows_shard_picks(cfg)
    t0 = time.time()
    import pickle

    cache = Path(f"/tmp/rows_shard_c{cfg}.pkl")   # scratch: reruns skip the shards
    if cache.exists():
        outs = pickle.loads(cache.read_bytes())
    else:
        with mp.get_context("fork").Pool(SHARD_WORKERS) as pool:
            outs = pool.map(_shard_worker, [(cfg, sh) for sh in shards])
        cache.write_bytes(pickle.dumps(outs))
    p, img, net, conv = _shard_setup(cfg)
    fp = R_fv.FvParams.from_backend(p)
    q = [int(x) for x in fp.q_primes]
    qcol = np.asarray(q, dtype=np.int64)[:, None]
    n_out = len(outs[0]["parts"])
    summed = []
    for m in range(n_out):
        parts = []
        for c in range(2):
            acc = np.zeros_like(outs[0]["parts"][m][c])
            for o in outs:
                acc = (acc + o["parts"][m][c]) % qcol
            parts.append(acc)
        summed.append(parts)
    out = {"config": cfg, "key_seed": 1234, "total_rows": total, "picks": picks,
           "shards": shards, "workers": SHARD_WORKERS,
           "shard_enc": outs[0]["enc"],
           "shard_levels": outs[0]["levels"],
           "shard_costs": [o["cost"] for o in outs],
           "shard_seconds": [o["seconds"] for o in outs],
           "conv_out": [digest(parts) for parts in summed]}
    assert all(o["enc"] == outs[0]["enc"] for o in outs)
    # the reference's own square (and FC) on the summed layer output
    be = R_fv.FvBackend(p, rng=np.random.default_rng(1234))
    pv = R_inf.pack_image(be, img)
    assert [digest(ct.parts) for ct in pv.cts] == outs[0]["enc"]
    lvl = outs[0]["levels"][0]
    cts = [R_fv.FvCiphertext([np.asarray(x) for x in parts], lvl, be.params)
           for parts in summed]
    x = R_inf.PackedVector(total, pv.slots_used, cts)
    t1 = time.time()
    sq = R_inf.square_activation(be, x)
    out["square_out"] = [digest(ct.parts) for ct in sq.cts]
    out["square_levels"] = [ct.level_used for ct in sq.cts]
    if cfg == 2:
        fc = net.layers[2]
        rows = R_inf.compile_fc(fc, sq.slots_used)
        res = R_inf.layer_eval(be, rows, sq)
        out["fc_out"] = [digest(ct.parts) for ct in res.cts]
        out["fc_levels"] = [ct.level_used for ct in res.cts]
        out["logits"] = [int(v) for v in R_inf.decrypt_logits(be, res)]
        # the same square / FC over the summed input, decrypted slot values
        out["square_dec_digest"] = [vec_digest(be.decrypt(ct)) for ct in sq.cts]
    out["tail_seconds"] = time.time() - t1
    out["seconds"] = time.time() - t0
    dump(f"rows_shard_c{cfg}.json", out)


if __name__ == "__main__" and "--rows-shard" in sys.argv:
    for c in (2, 3):
        if f"--c{c}" in sys.argv or not any(f"--c{x}" in sys.argv for x in (2, 3)):
            gen_rows_shard(c)


# ---- config 4: the 50-62-bit key switch, run by the reference -------------
KS64_CASES = [(4096, 2), (4096, 4), (4096, 8), (16384, 2), (16384, 4), (16384, 8), (65536, 2)]


def _ks64_one(args):
    n, L = args
    primes = R_ntt.find_ntt_primes(L, 60, 2 * n)
    t = R_ntt.find_ntt_primes(1, 20, 2 * n)[0]
    ctx = R_fv._FvContext(R_fv.FvParams(n=n, t=t, q_primes=primes))
    seed = 4000 + n + L
    rng = np.random.default_rng(seed)
    t0 = time.time()
    s = ctx.to_rns(ctx.rand_ternary(rng))
    key = R_fv._keyswitch_key(ctx, s, ctx.mul(s, s), rng)
    c = ctx.rand_uniform(rng)
    t1 = time.time()
    d0, d1 = R_fv._keyswitch_apply(ctx, c, key)
    t2 = time.time()
    return {"n": n, "L": L, "bits": 60, "primes": primes, "t": t, "seed": seed,
            "key": key_digest(key), "c": digest([c]), "d0": digest([d0]), "d1": digest([d1]),
            "keygen_seconds": t1 - t0, "apply_seconds": t2 - t1}


def gen_ks64():
    """Reference _keyswitch_key + _keyswitch_apply (fv.py:176-217) over
    _FvContext(FvParams(n, t, 60-bit primes)) -- the object-dtype path."""
    import multiprocessing as mp

    with mp.get_context("fork").Pool(len(KS64_CASES)) as pool:
        cases = pool.map(_ks64_one, KS64_CASES)
    dump("ks64.json", {"cases": cases})


if __name__ == "__main__" and "--ks64" in sys.argv:
    gen_ks64()


def gen_config5_enc_impl(count=3, image_seed=5):
    """Config 5: the first images of the stream (configs.batch_images: one
    default_rng(5) drawing (1, 96, 96) images in turn) encrypted in sequence
    under one key -- one Generator for keygen and every encryption."""
    rng = np.random.default_rng(image_seed)
    imgs = [rng.integers(0, 256, (1, 96, 96), dtype=np.int64) for _ in range(count)]
    be = R_fv.FvBackend(profile("retina"), rng=np.random.default_rng(1234))
    enc = [[digest(ct.parts) for ct in R_inf.pack_image(be, img).cts] for img in imgs]
    dump("config5_enc.json", {"key_seed": 1234, "image_seed": image_seed, "enc": enc})


if __name__ == "__main__" and "--config5" in sys.argv:
    gen_config5_enc_impl()
