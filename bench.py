"""Benchmark: encrypted-image inference latency of BASELINE.json's config 2
(ROP-shaped 96x96x1 net at the reference's 80-bit `retina` profile) on
B200, plus the RNS-NTT polys/sec microbench (config 4) as a secondary.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one full encrypted inference of one image through the
reference-compatible API.  `value` times the device-resident step:
`infer(backend, net, pv)` on an already-encrypted image in HBM.  `e2e`
times the public-API path from host pixels to host logits:
`pack_image` (host->device) + `infer` + `decrypt_logits` (device->host).
Every step's working set (888 MB of switch keys, GBs of row tiles) exceeds
the 126 MB L2, so no explicit flush is needed.

Multi-GPU: the path does not shard (north star: one GPU); N ranks run N
independent replicas, timed as the max over ranks, `scaling: "weak"`.

--impl reference times the reference algorithm on the host CPU (the oracle
port, oracle/fv_oracle.py, with all host cores) on a bounded sample per
step, extrapolated to one image with the exact serial op counts.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "encrypted-image inference latency (ms) & RNS-NTT polys/sec, 1 B200"
CONFIG = {"workload": "config2: ROP-shaped CaRENet, 96x96x1 image, conv 5x5x5 stride 2, square, "
                      "fc 10580->2; profile retina (N=16384, 22 x 30-bit q primes, "
                      "t=4503599627763713)", "batch": 1,
          "data": "synthetic: pixels/weights default_rng(2), keys+encryption default_rng(1234)",
          "l2": "working set > L2 (888 MB keys, multi-GB row tiles); no flush needed"}


def _env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, val in zip(names, r[3:7]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(value, world, device="cuda"):
    """Max of a per-rank timing over all ranks (NCCL on the GPU, gloo in tests)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _ks_work(ctx) -> dict:
    """Algorithmic work of one key switch of one ciphertext.

    Reference formulation (fv.py:205-217): M = (k^2 + 2k)
    ((N/2) log2 N + N) + 2 k^2 N modmuls.  The aux-basis key switch that runs
    here (ks_aux.cu) computes the same limbs with 3k forward + 6k inverse
    transforms of (N/2) log2 N butterflies, a 3 * 2k * k * N multiply-add
    contraction and a 6-modmul CRT per output coefficient (2kN of them)."""
    k, n = ctx.k, ctx.n
    logn = n.bit_length() - 1
    ref = (k * k + 2 * k) * ((n // 2) * logn + n) + 2 * k * k * n
    out = {"modmuls": ref, "key_bytes": 2 * k * k * n * 4, "ct_bytes": 3 * k * n * 4,
           "aux": bool(getattr(ctx, "ks_aux", False))}
    if out["aux"]:
        out.update(butterflies=9 * k * (n // 2) * logn, macs=6 * k * k * n, crt_modmuls=12 * k * n,
                   key_bytes=6 * k * k * n * 4,
                   # digits in (k rows), X out + in (3k + 3k), Y out + in (6k + 6k), 2k rows out
                   ct_bytes=21 * k * n * 4)
    return out


def run_ours(args, rank, local_rank, world):
    import numpy as np
    import torch

    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200 import inference as I
    from paper_1901_10074_b200 import planner
    from paper_1901_10074_b200.configs import (KEY_SEED, config_network, config_params,
                                               workload_op_counts)
    from paper_1901_10074_b200.fv import FvBackend

    cfg = args.config
    img, net = config_network(cfg)
    params = config_params(cfg)
    t_setup = time.perf_counter()
    be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t_setup
    pv = I.pack_image(be, img)
    torch.cuda.synchronize()

    def device_step():
        out = I.infer(be, net, pv)
        return out

    # ---- warm-up
    for _ in range(args.warmup):
        out = device_step()
    torch.cuda.synchronize()
    _barrier(world)

    # ---- timed region: device-resident step, KS launches bracketed by events
    planner.KS_EVENTS = []
    launches0 = nat.launch_count()
    ks0 = dict(planner.STATS)
    clocks = ClockSampler(local_rank)
    clocks.start()
    torch.cuda.synchronize()
    _barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        out = device_step()
    e1.record()
    torch.cuda.synchronize()
    _barrier(world)
    clk = clocks.stop()
    step_ms = e0.elapsed_time(e1) / args.steps
    launches = (nat.launch_count() - launches0) / args.steps
    ks_events = planner.KS_EVENTS
    planner.KS_EVENTS = None
    ks_ms = sum(a.elapsed_time(b) for a, b, _ in ks_events)
    ks_cts = sum(bt for _, _, bt in ks_events)
    ks_launches = len(ks_events)
    del ks0
    logits = I.decrypt_logits(be, out)
    step_ms = _max_over_ranks(step_ms, world)

    # ---- e2e through the public API with host buffers
    for _ in range(1):
        I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    torch.cuda.synchronize()
    nat.TRAFFIC["h2d"] = nat.TRAFFIC["d2h"] = 0
    _barrier(world)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        lg = I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    e3.record()
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks(e2.elapsed_time(e3) / args.steps, world)
    h2d = nat.TRAFFIC["h2d"] / args.steps
    d2h = nat.TRAFFIC["d2h"] / args.steps

    result = None
    if rank == 0:
        # correctness: decrypted logits equal the exact plaintext forward pass mod t
        from paper_1901_10074_b200.configs import centred_mod, plaintext_forward

        want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
        ok = [int(v) for v in logits] == want and [int(v) for v in lg] == want
        # integer-pipe peak (measured on this GPU) and the KS roofline
        peak = _int_peak()
        work = _ks_work(be.ctx)
        avg_launch_ms = ks_ms / max(1, ks_launches)
        cts_per_launch = ks_cts / max(1, ks_launches)
        t_ct = avg_launch_ms * 1e-3 / max(1e-9, cts_per_launch)  # seconds per key switch
        bf_peak = peak["shoup_butterfly"]
        traffic = _ncu_traffic(cts_per_launch, work["aux"])
        counts = workload_op_counts(cfg)
        hbm = {"algorithmic_bytes_per_launch": int(work["key_bytes"] + work["ct_bytes"]
                                                   * cts_per_launch),
               "achieved_GBs": round((work["key_bytes"] + work["ct_bytes"] * cts_per_launch)
                                     / (avg_launch_ms * 1e-3) / 1e9, 1),
               "peak_GBs": _hbm_peak()}
        common = {"avg_launch_ms": round(avg_launch_ms, 4),
                  "cts_per_launch": round(cts_per_launch, 1),
                  "launches_in_step": ks_launches / args.steps,
                  "ks_share_of_step": round(ks_ms / args.steps / step_ms, 4),
                  "traffic": traffic, "hbm_view": hbm,
                  "reference_formulation_Tmodmul_s": round(work["modmuls"] / t_ct / 1e12, 3)}
        if work["aux"]:
            # butterfly-equivalent ops: transforms + CRT at the butterfly rate,
            # the contraction at the measured 32x32->64 multiply (IMAD.WIDE) rate
            equiv = (work["butterflies"] + work["crt_modmuls"]
                     + work["macs"] * bf_peak / peak["imad_wide"])
            achieved = equiv / t_ct / 1e12
            roofline = {
                "kernel": "aux-basis key switch: k_ksa_fwd (3k NTTs) -> k_ksa_mac (64-bit "
                          "contraction) -> k_ksa_inv (6k iNTTs + exact CRT)",
                "bound": "int-pipe (IMAD)", "unit": "Tmodmul/s (butterfly-equivalent)",
                "achieved": round(achieved, 3), "peak": round(bf_peak, 3),
                "frac": round(achieved / bf_peak, 4),
                "peak_source": "measured live by tools/probe_int: lazy Shoup butterfly "
                               f"{bf_peak:.2f} T/s, IMAD.WIDE {peak['imad_wide']:.2f} T/s",
                "work_per_ct": (f"{work['butterflies']} butterflies (9k transforms) + "
                                f"{work['macs']} multiply-adds (6k^2 N) + {work['crt_modmuls']} "
                                "CRT modmuls"),
                "ideal_us_per_ct": round(equiv / bf_peak / 1e6, 3),
                "measured_us_per_ct": round(t_ct * 1e6, 3), **common}
        else:
            achieved = work["modmuls"] / t_ct / 1e12
            roofline = {
                "kernel": "k_keyswitch<14,4> (fused digit NTT -> MAC -> iNTT)",
                "bound": "int-pipe (IMAD)", "unit": "Tmodmul/s",
                "achieved": round(achieved, 3), "peak": round(bf_peak, 3),
                "frac": round(achieved / bf_peak, 4),
                "peak_source": "measured live by tools/probe_int (lazy Shoup butterfly = 1 modmul "
                               "+ 3 adds, 8 independent chains/thread, whole GPU)",
                "work_per_ct": f"(k^2+2k)((N/2)log2N+N)+2k^2N = {work['modmuls']} modmuls",
                **common}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = _cpu_baseline_single(params, counts)
        ntt = None if args.no_ntt else _ntt_microbench(peak)
        result = {
            "metric": METRIC, "value": round(step_ms, 3), "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_ms, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 (30-bit RNS limbs), u64 plaintext", "data": "synthetic",
            "config": dict(CONFIG, parallelism=f"replicas x{world}" if world > 1 else "single GPU"),
            "images_per_s": round(world * 1000.0 / step_ms, 4),
            "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "pack_image(host pixels) + infer + decrypt_logits(host logits)"},
            "gpu_launches": int(round(launches)),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
            "correct": ok,
            "op_counts_per_image": counts,
            "keygen_s": round(keygen_s, 2),
            "ntt_microbench": ntt,
        }
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return result


def _int_peak() -> dict:
    import torch

    sys.path.insert(0, str(ROOT / "tools"))
    from probe_int import measure

    names = ["imad", "imad_hi", "imad_wide", "iadd3", "shoup_butterfly", "shoup_butterfly64"]
    out = {n: measure(k) / 1e12 for k, n in enumerate(names) if n != "iadd3"}
    torch.cuda.synchronize()
    return out


def _hbm_peak():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        return 6650.0


def _ncu_traffic(cts_per_launch=None, aux=False):
    """dram bytes (read + write) per key-switch launch from the committed ncu
    capture (profiles/ks_aux_traffic.json for the aux-basis kernels,
    profiles/ks_traffic.json for k_keyswitch), scaled to this run's launch."""
    p = ROOT / "profiles" / ("ks_aux_traffic.json" if aux else "ks_traffic.json")
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
    except Exception:
        return None
    per_ct = d.get("dram_bytes_per_ct")
    if per_ct is None or cts_per_launch is None:
        return d.get("dram_bytes_per_launch")
    return int(per_ct * cts_per_launch)


def _cpu_baseline_single(params, counts) -> dict:
    from oracle import cpu_baseline as cb

    t0 = time.perf_counter()
    per_op = cb.time_ops(params, hops=6, cmults=3)
    sec = cb.extrapolate(per_op, counts, workers=1)
    return {"value": round(sec * 1000.0, 1), "unit": "ms", "cores": 1, "kind": "port",
            "sample": "oracle (CPU restatement of hepack fv/ntt, C butterflies) at retina: "
                      "6 key-switch hops, 3 ct x pt, 10 adds, 1 square+relin, 1 encrypt, "
                      "1 decrypt; per-image latency extrapolated with the exact serial op "
                      f"counts {counts}",
            "per_op_s": {k: round(v, 4) for k, v in per_op.items()},
            "wall_s": round(time.perf_counter() - t0, 1)}


def _ntt_microbench(peaks=None):
    """Config 4 secondary: batched forward/inverse NTT polys/s (device order),
    with each entry's roofline fraction: per-limb work (N/2) log2 N + N
    modmuls against the measured lazy Shoup butterfly rate of
    the word size (32-bit or 64-bit)."""
    import ctypes as C

    import torch

    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity

    lib = nat.load()
    res, fracs = {}, {}
    for log_n, bits, L, batch in [(16, 60, 8, 64), (15, 55, 8, 128), (14, 60, 8, 256),
                                  (13, 60, 8, 256), (12, 50, 8, 1024), (14, 30, 22, 256)]:
        n = 1 << log_n
        primes = find_ntt_primes(L, bits, 2 * n)
        psis = [root_of_unity(p, n) for p in primes]
        h = C.c_void_p()
        wide = bits > 30
        if wide:
            nat.check(lib.hefv_ctx_create(C.byref(h), log_n, 0, None, None, L,
                                          (C.c_uint64 * L)(*primes), (C.c_uint64 * L)(*psis)))
            x = torch.randint(0, 1 << 40, (batch, L, n), dtype=torch.int64, device="cuda")
            f, g = lib.hefv_ntt_fwd64, lib.hefv_ntt_inv64
        else:
            nat.check(lib.hefv_ctx_create(C.byref(h), log_n, L, (C.c_uint32 * L)(*primes),
                                          (C.c_uint32 * L)(*psis), 0, None, None))
            x = torch.randint(0, 1 << 29, (batch, L, n), dtype=torch.int32, device="cuda")
            f, g = lib.hefv_ntt_fwd32, lib.hefv_ntt_inv32
        y = torch.empty_like(x)
        st = torch.cuda.current_stream().cuda_stream
        for fn, name in ((f, "fwd"), (g, "inv")):
            src = x if name == "fwd" else y
            dst = y if name == "fwd" else x
            nat.check(fn(h, src.data_ptr(), dst.data_ptr(), batch, L, 0, 0, st))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                nat.check(fn(h, src.data_ptr(), dst.data_ptr(), batch, L, 0, 0, st))
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            ps = batch * L / (ms * 1e-3)
            key = f"N=2^{log_n},{bits}-bit,L={L},batch={batch},{name}"
            res[key] = round(ps, 1)
            if peaks:
                pk = peaks["shoup_butterfly64" if wide else "shoup_butterfly"]
                tm = ps * ((n // 2) * log_n + n) / 1e12
                fracs[key] = {"Tmodmul_s": round(tm, 3), "peak": round(pk, 3),
                              "frac": round(tm / pk, 3)}
        lib.hefv_ctx_destroy(h)
    out = {"unit": "limb-polys/s", **res}
    if peaks:
        out["roofline"] = fracs
    out["keyswitch64"] = _ks64_microbench(peaks)
    return out


def _ks64_microbench(peaks=None):
    """Config 4: a full key switch over L = 8 60-bit primes (the reference's
    _keyswitch_apply, fv.py:205-217), ciphertexts/s; roofline in the
    reference formulation's (L^2 + 2L)((N/2) log2 N + N) + 2 L^2 N modmuls per
    ciphertext against the measured 64-bit butterfly rate."""
    import torch

    from paper_1901_10074_b200.ring import find_ntt_primes
    from paper_1901_10074_b200.rns import RnsKeySwitch64

    out = {"unit": "us per ciphertext"}
    for log_n, L, B in [(14, 8, 32), (16, 8, 8)]:
        n = 1 << log_n
        ks = RnsKeySwitch64(find_ntt_primes(L, 60, 2 * n), n)
        key = ks.random_key(1)
        p = torch.tensor(ks.primes, dtype=torch.int64, device="cuda").view(1, L, 1)
        dig = torch.randint(0, 1 << 62, (B, L, n), dtype=torch.int64, device="cuda") % p
        ks.switch(key, dig)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            ks.switch(key, dig)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 3 / B * 1e3
        mm = (L * L + 2 * L) * ((n // 2) * log_n + n) + 2 * L * L * n
        ent = {"us_per_ct": round(us, 2), "path": "aux" if ks.aux else "direct",
               "ref_Tmodmul_s": round(mm / us / 1e6, 3)}
        if peaks:
            ent["frac_of_64bit_butterfly_peak"] = round(mm / us / 1e6 / peaks["shoup_butterfly64"], 3)
        out[f"N=2^{log_n},60-bit,L={L},B={B}"] = ent
        del ks
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on the host CPU (oracle port)
# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return None
    from oracle import cpu_baseline as cb
    from paper_1901_10074_b200.configs import config_params, workload_op_counts

    params = config_params(args.config)
    counts = workload_op_counts(args.config)
    workers = cb.physical_cores()
    vals = []
    t_all = time.perf_counter()
    state = cb.prepare(params)
    for i in range(args.warmup + args.steps):
        per_op = cb.time_ops_parallel(state, workers, hops=2, cmults=1)
        if i >= args.warmup:
            vals.append(cb.extrapolate(per_op, counts, workers=workers) * 1000.0)
    value = statistics.mean(vals) if vals else float("nan")
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "ms", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value, 1), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64 numpy residues", "data": "synthetic",
        "config": dict(CONFIG, parallelism=f"{workers} CPU processes"),
        "cpu_baseline": {"value": round(value, 1), "unit": "ms", "cores": workers, "kind": "port",
                         "sample": "per step, every core runs 2 key-switch hops, 1 ct x pt, "
                                   "10 adds, 1 square+relin, 1 encrypt, 1 decrypt at retina; "
                                   "per-image latency = sum_op count x time / cores with the "
                                   f"exact serial counts {counts}"},
        "e2e": {"value": round(value, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_all, 1),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ntt", action="store_true")
    args = ap.parse_args()
    rank, local_rank, world = _env_rank()
    if args.warmup < 1:
        args.warmup = 1
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, local_rank, world)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
