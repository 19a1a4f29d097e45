"""CPU BASELINE -- the reference itself (hepack + numba) timed on the host.
BENCH INFRASTRUCTURE ONLY: bench.py's cpu_baseline leg and its
``--impl reference`` arm import this module; the product never does.

The reference is installed unmodified in ``baseline/_ref`` (git-ignored; it
travels to the GPU box with the snapshot; recipe in DESIGN.md "Reference
install").  Whole encrypted images take the reference 30+ hours per core at
retina, so a run times a bounded sample of the reference's own operations
on its own FvBackend -- key-switch hops (``rotate`` by a key offset: Galois
automorphism + ``_keyswitch_apply``, fv.py:417-432), ct x pt products
(``_cmult``), additions, one ct x ct square with relinearisation
(``_mult``), one encryption and one decryption -- and extrapolates with the
exact serial op counts of the config (configs.workload_op_counts):

    latency(image) = sum_op count(op) * t(op)          one process

The reference is serial per image; P worker processes running whole images
give images/s = P / latency(image measured while all P run).

Keys: the ``--impl reference`` arm generates them with the reference's own
keygen (untimed setup).  The ours-arm leg, limited to ~30 s of CPU, builds
the reference's KeySet from the GPU keygen's output instead (bit-identical
to the reference's keygen from the same seed: tests/test_gpu_ops.py,
tests/golden/retina.json) and only with the keys the sample uses.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


def load_hepack():
    """The installed reference package, or None when it is not installed."""
    if not (REF / "hepack" / "__init__.py").exists():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import hepack
    import hepack.fv
    import hepack.inference
    import hepack.ntt  # noqa: F401

    return hepack


def cpu_info() -> dict:
    """CPU model, logical CPUs available to this process, physical cores."""
    model, phys = None, set()
    cur = {}
    try:
        for line in open("/proc/cpuinfo"):
            if ":" not in line:
                if "physical id" in cur and "core id" in cur:
                    phys.add((cur["physical id"], cur["core id"]))
                cur = {}
                continue
            k, v = (x.strip() for x in line.split(":", 1))
            cur[k] = v
            if k == "model name" and model is None:
                model = v
        if "physical id" in cur and "core id" in cur:
            phys.add((cur["physical id"], cur["core id"]))
    except OSError:
        pass
    try:
        logical = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        logical = os.cpu_count() or 1
    physical = min(len(phys), logical) if phys else logical
    return {"model": model, "logical": logical, "physical": physical}


def ref_params(H, cfg: int):
    p = H.params.profile("desk" if cfg == 1 else "retina")
    if cfg == 3:
        p = p.replace(coeff_modulus_bits=720)
    return p


def keyset_from_gpu(H, gpu_keys, offsets=(1,)):
    """The reference's KeySet (fv.py:220-228) holding the GPU keygen's keys
    in the reference's stored form (natural-order NTT stacks)."""
    fp_g = gpu_keys.context.fp
    fp = H.fv.FvParams(n=fp_g.n, t=fp_g.t, q_primes=list(fp_g.q_primes), sigma=fp_g.sigma)
    ctx = H.fv._FvContext(fp)
    sk = lambda k: H.fv.SwitchKey(body=list(k.body), mask=list(k.mask))  # noqa: E731
    return H.fv.KeySet(context=ctx, secret=gpu_keys.secret, public=tuple(gpu_keys.public),
                       relin=sk(gpu_keys.relin),
                       galois={off: sk(gpu_keys.galois[off]) for off in offsets})


def reference_backend(H, cfg: int, keys=None, seed=1234):
    """The reference's FvBackend; ``keys=None`` runs its own keygen."""
    return H.fv.FvBackend(ref_params(H, cfg), keys=keys, rng=np.random.default_rng(seed))


def prepare(be):
    rng = np.random.default_rng(99)
    t = be.params.plain_modulus
    vec = rng.integers(0, min(t, 1 << 62), be.params.slot_count)
    c = time.perf_counter()
    ct = be.encrypt(vec)
    return {"be": be, "vec": vec, "ct": ct, "t_encrypt": time.perf_counter() - c}


def sample(state, hops=1, cmults=1, adds=10) -> dict:
    """Per-op seconds of the reference's own operations on this core."""
    be, vec, ct = state["be"], state["vec"], state["ct"]
    res = {}
    cur = ct
    if hops:
        c = time.perf_counter()
        for _ in range(hops):
            cur = be.rotate(cur, 1)      # one hop: a Galois key for offset 1 exists
        res["ks_hop"] = (time.perf_counter() - c) / hops
    if cmults:
        c = time.perf_counter()
        for _ in range(cmults):
            be.cmult(ct, vec)
        res["cmult"] = (time.perf_counter() - c) / cmults
    if adds:
        c = time.perf_counter()
        for _ in range(adds):
            be.add(ct, cur)
        res["add"] = (time.perf_counter() - c) / adds
    return res


def sample_heavy(state, t_hop: float) -> dict:
    """Square with relinearisation (tensor part = mult - one hop), decrypt."""
    be, ct = state["be"], state["ct"]
    c = time.perf_counter()
    sq = be.mult(ct, ct)
    t_mult = time.perf_counter() - c
    c = time.perf_counter()
    be.decrypt(sq)
    t_dec = time.perf_counter() - c
    return {"mult_tensor": max(0.0, t_mult - t_hop), "decrypt": t_dec,
            "encrypt": state["t_encrypt"]}


def extrapolate(per_op: dict, counts: dict) -> float:
    """Seconds per image (one process) from per-op times and exact counts."""
    return (counts["ks_hops"] * per_op["ks_hop"] + counts["cmult"] * per_op["cmult"]
            + counts["add"] * per_op["add"] + counts["mult"] * per_op["mult_tensor"]
            + counts["encrypt"] * per_op["encrypt"]
            + counts.get("decrypt", 1) * per_op["decrypt"])


_STATE = None


def _worker(args):
    return sample(_STATE, *args)


def sample_parallel(state, workers: int, hops=1, cmults=1, adds=10) -> list:
    """The light sample run by ``workers`` forked processes at once (the
    prepared backend shared copy-on-write); per-worker per-op seconds."""
    import multiprocessing as mp

    global _STATE
    _STATE = state
    with mp.get_context("fork").Pool(workers) as pool:
        return pool.map(_worker, [(hops, cmults, adds)] * workers)


def ntt_object_path(H, sizes=(12, 13, 14, 15, 16), bits=60, reps=1) -> dict:
    """Config 4 on the reference: NttPrime(p, N).fwd / inv for one ~60-bit
    prime (the object-dtype path, ntt.py:202-224), limb-polys/s per size."""
    out = {}
    rng = np.random.default_rng(4)
    for log_n in sizes:
        n = 1 << log_n
        p = H.ntt.find_ntt_primes(1, bits, 2 * n)[0]
        tr = H.ntt.NttPrime(p, n)
        a = np.array([int(v) for v in rng.integers(0, p, n, dtype=np.uint64)], dtype=object)
        c = time.perf_counter()
        for _ in range(reps):
            ev = tr.fwd(a)
        t_f = (time.perf_counter() - c) / reps
        c = time.perf_counter()
        for _ in range(reps):
            tr.inv(ev)
        t_i = (time.perf_counter() - c) / reps
        out[f"N=2^{log_n},{bits}-bit,fwd"] = round(1.0 / t_f, 2)
        out[f"N=2^{log_n},{bits}-bit,inv"] = round(1.0 / t_i, 2)
    return out


def reference_network(H, cfg: int):
    """The reference's own NetworkSpec objects for a config (the draws of
    configs.config_network)."""
    from paper_1901_10074_b200.configs import config_network

    img, net = config_network(cfg)
    R = H.inference
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


def config1_full(H, seed=1234) -> dict:
    """Config 1 measured IN FULL on one core: the reference's own keygen
    (untimed), then pack_image -> infer -> decrypt_logits exactly as its CLI
    runs them (inference.py:178-452; cli.py:151-155)."""
    img, net = reference_network(H, 1)
    t0 = time.perf_counter()
    be = reference_backend(H, 1, seed=seed)
    keygen = time.perf_counter() - t0
    t1 = time.perf_counter()
    logits = H.inference.decrypt_logits(be, H.inference.infer(be, net, H.inference.pack_image(
        be, img)))
    ms = (time.perf_counter() - t1) * 1000.0
    return {"ms": round(ms, 1), "keygen_s": round(keygen, 2),
            "logits": [int(v) for v in logits]}
