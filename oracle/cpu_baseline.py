"""ORACLE -- CPU baseline timing of the reference algorithm. TEST/BENCH INFRASTRUCTURE.

Times the CPU restatement of the reference's FV path (oracle/fv_oracle.py,
numpy + C butterflies in place of numba) on a bounded sample of a config's
operations and extrapolates the per-image latency with the exact serial
op counts (SURVEY.md 8d "CPU baseline"):

    latency = sum_op count(op) * t(op)      (one core; / P with P workers)

The sample: key-switch hops (Galois automorphism + RNS-limb key switch, the
~85 % term), ct x pt products, additions, one ct x ct square with
relinearisation, one encryption and one decryption.  Only bench.py's CPU
legs import this module.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import fv_oracle as O


def _setup(params, seed=1234):
    fp = O.OracleParams.from_backend(params)
    rng = np.random.default_rng(seed)
    ctx = O.OracleContext(fp)
    s = ctx.rns(ctx.rand_ternary(rng))
    a = ctx.rand_uniform(rng)
    e = ctx.rns(ctx.rand_error(rng))
    pk = ((-(ctx.ring_mul(a, s) + e)) % ctx.pcol, a)
    relin = O.switch_key(ctx, s, ctx.ring_mul(s, s), rng)
    g1 = O.switch_key(ctx, s, ctx.galois(s, pow(3, 1, 2 * fp.n)), rng)
    keys = O.OracleKeys(ctx, s, pk, relin, {1: g1})
    be = O.OracleFvBackend(params, keys=keys, rng=rng)
    return be, rng


def prepare(params, seed=1234):
    """Context, two switch keys (relin + Galois offset 1), a fresh ciphertext."""
    t0 = time.perf_counter()
    be, rng = _setup(params, seed)
    t = params.plain_modulus
    vec = rng.integers(0, min(t, 1 << 62), params.slot_count)
    c = time.perf_counter()
    ct = be.encrypt(vec)
    t_enc = time.perf_counter() - c
    return {"be": be, "vec": vec, "ct": ct, "t_encrypt": t_enc,
            "setup_seconds": time.perf_counter() - t0}


def sample(state, hops=6, cmults=3) -> dict:
    """Per-op seconds on this core, on a prepared state."""
    be, vec, ct = state["be"], state["vec"], state["ct"]
    res = {"encrypt": state["t_encrypt"]}
    c = time.perf_counter()
    cur = ct
    for _ in range(hops):
        cur = be.rotate(cur, 1)
    res["ks_hop"] = (time.perf_counter() - c) / hops
    c = time.perf_counter()
    for _ in range(cmults):
        be.cmult(ct, vec)
    res["cmult"] = (time.perf_counter() - c) / cmults
    c = time.perf_counter()
    for _ in range(10):
        be.add(ct, cur)
    res["add"] = (time.perf_counter() - c) / 10
    c = time.perf_counter()
    sq = be.mult(ct, ct)
    res["mult_tensor"] = max(0.0, time.perf_counter() - c - res["ks_hop"])  # relin = 1 hop
    c = time.perf_counter()
    be.decrypt(sq)
    res["decrypt"] = time.perf_counter() - c
    return res


def time_ops(params, hops=6, cmults=3, seed=1234) -> dict:
    state = prepare(params, seed)
    res = sample(state, hops, cmults)
    res["setup_seconds"] = state["setup_seconds"]
    return res


def extrapolate(per_op: dict, counts: dict, workers: int = 1) -> float:
    """Seconds per image from per-op times and the exact serial op counts."""
    total = (counts["ks_hops"] * per_op["ks_hop"] + counts["cmult"] * per_op["cmult"]
             + counts["add"] * per_op["add"] + counts["mult"] * per_op["mult_tensor"]
             + counts["encrypt"] * per_op["encrypt"] + counts.get("decrypt", 1) * per_op["decrypt"])
    return total / workers


_STATE = None


def _worker(args):
    hops, cmults = args
    return sample(_STATE, hops, cmults)


def time_ops_parallel(state, workers: int, hops=2, cmults=1):
    """Per-op times measured while `workers` forked processes (sharing the
    prepared state copy-on-write) run the sample concurrently."""
    import multiprocessing as mp

    global _STATE
    _STATE = state
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        results = pool.map(_worker, [(hops, cmults)] * workers)
    return {k: float(np.mean([r[k] for r in results])) for k in results[0]}


def physical_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
