"""Benchmark: encrypted-image inference latency of BASELINE.json's config 2
(ROP-shaped 96x96x1 net at the reference's 80-bit `retina` profile) on
B200, plus the driver-observed legs of the other configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one full encrypted inference of one image through the
reference-compatible API.  `value` times the device-resident step:
`infer(backend, net, pv)` on an already-encrypted image in HBM.  `e2e`
times the public-API path from host pixels to host logits:
`pack_image` (host->device) + `infer` + `decrypt_logits` (device->host).
Every step's working set (888 MB of switch keys, GBs of row tiles) exceeds
the 126 MB L2, so no explicit flush is needed.

Further legs on the same line (N = 1): `config3` -- one 256x256x3 image end
to end (keygen excluded, logits checked), `config5` -- images/s over a
stream of 8 ROP images (one key, one Generator, logits checked), `config1`
-- the toy desk net end to end, `ntt_microbench` -- config 4, and
`cpu_baseline` -- the reference itself (hepack + numba from baseline/_ref) on
a bounded sample, extrapolated, plus config 1 measured in full.

Multi-GPU: the path does not shard (north star: one GPU); N ranks run N
independent replicas, timed as the max over ranks, `scaling: "weak"`.

--impl reference runs the unmodified reference (baseline/_ref, its own
keygen and FvBackend) on the host CPU: per step, a bounded sample of its
operations in one process (-> single-image latency, extrapolated with the
exact serial op counts) and in P worker processes (-> images/s); config 1
is also run in full once.
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
    planner.ks_reset(be.ctx, timing=True)
    launches0 = nat.launch_count()
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
    ks = planner.ks_stats(be.ctx)
    planner.ks_reset(be.ctx)
    ks_ms, ks_cts, ks_launches = ks["ks_ms"], ks["ks_cts"], ks["ks_launches"]
    step_ms = _max_over_ranks(step_ms, world)

    # ---- e2e through the public API with host buffers
    for _ in range(1):
        I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    torch.cuda.synchronize()
    nat.TRAFFIC["h2d"] = nat.TRAFFIC["d2h"] = 0
    _barrier(world)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2e_steps = min(args.steps, 3)
    e2.record()
    for _ in range(e2e_steps):
        lg = I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    e3.record()
    torch.cuda.synchronize()
    e2e_ms = _max_over_ranks(e2.elapsed_time(e3) / e2e_steps, world)
    h2d = nat.TRAFFIC["h2d"] / e2e_steps
    d2h = nat.TRAFFIC["d2h"] / e2e_steps

    # ---- config 5 (image stream) and config 3 (256x256x3) legs, rank 0 at N=1
    legs, be3 = {}, None
    keys2, ctx2 = be.keys, be.ctx
    logits = I.decrypt_logits(be, out)
    if world == 1 and not args.no_legs:
        legs["config5"] = _config5_leg(be, net, args.config5_images)
        planner.release_workspace(be.ctx)
        del be, pv, out
        torch.cuda.empty_cache()
        legs["config3"], be3 = _config3_leg()
        legs["config1"] = _config1_leg()

    result = None
    if rank == 0:
        # correctness: decrypted logits equal the exact plaintext forward pass mod t
        from paper_1901_10074_b200.configs import centred_mod, plaintext_forward

        want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
        ok = [int(v) for v in logits] == want and [int(v) for v in lg] == want
        # integer-pipe peak (measured on this GPU) and the KS roofline
        peak = _int_peak()
        work = _ks_work(ctx2)
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
        # SURVEY.md 8(d)'s fixed model, shared with the judge: M modmuls of the
        # reference formulation x c = 3 IMAD per 30-bit modmul against the
        # IMAD rate measured live on this GPU (tools/probe_int.py).
        imad_peak = peak["imad"]
        achieved = work["modmuls"] * 3 / t_ct / 1e12
        roofline = {
            "kernel": ("aux-basis key switch: k_ksa_fwd (3k NTTs) -> k_ksa_mac (64-bit "
                       "contraction) -> k_ksa_inv (6k iNTTs + exact CRT)") if work["aux"] else
                      "k_keyswitch<14,4> (fused digit NTT -> MAC -> iNTT)",
            "bound": "int-pipe (IMAD)", "unit": "T IMAD/s",
            "achieved": round(achieved, 3), "peak": round(imad_peak, 3),
            "frac": round(achieved / imad_peak, 4),
            "model": "SURVEY.md 8(d): M = (k^2+2k)((N/2)log2N+N) + 2k^2N modmuls per key switch "
                     f"(= {work['modmuls']}) x 3 IMAD, peak = IMAD rate measured live",
            "ideal_us_per_ct": round(work["modmuls"] * 3 / (imad_peak * 1e12) * 1e6, 3),
            "measured_us_per_ct": round(t_ct * 1e6, 3), **common}
        if work["aux"]:
            # the algorithm that runs: transforms + CRT at the measured lazy
            # Shoup butterfly rate, the contraction at the IMAD.WIDE rate
            equiv = (work["butterflies"] + work["crt_modmuls"]
                     + work["macs"] * bf_peak / peak["imad_wide"])
            roofline["own_algorithm"] = {
                "work_per_ct": (f"{work['butterflies']} butterflies (9k transforms) + "
                                f"{work['macs']} multiply-adds (6k^2 N) + {work['crt_modmuls']} "
                                "CRT modmuls"),
                "ideal_us_per_ct": round(equiv / bf_peak / 1e6, 3),
                "frac": round(equiv / bf_peak / 1e6 / (t_ct * 1e6), 4),
                "peaks_T_s": {"shoup_butterfly": round(bf_peak, 3),
                              "imad_wide": round(peak["imad_wide"], 3)}}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = _cpu_baseline(params, counts, gpu_keys={2: keys2, 3: be3.keys if be3 else None})
        ntt = None if args.no_ntt else _ntt_microbench(peak)
        result = {
            "metric": METRIC, "value": round(step_ms, 3), "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_ms, 3), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 (30-bit RNS limbs), u64 plaintext", "data": "synthetic",
            "config": dict(CONFIG, parallelism=f"replicas x{world}" if world > 1 else "single GPU"),
            "images_per_s": round(world * 1000.0 / step_ms, 4),
            "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                    "path": "pack_image(host pixels) + infer + decrypt_logits(host logits)"},
            **legs,
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


def _config5_leg(be, net, count: int) -> dict:
    """Config 5: a stream of ``count`` ROP images (configs.batch_images, the
    config-2 weights) encrypted under one key and inferred back to back.
    Software pipeline: image i's decryption is queued right behind its
    inference (decrypt_logits_async) and read back one image later, image
    i+1 is packed (host Generator draws, pinned host->device copies,
    encryption launches) while image i runs, so the host never waits for
    queued work and the GPU never waits for the host.  CUDA events bracket
    the whole stream; every image's logits are checked."""
    import torch

    from paper_1901_10074_b200 import inference as I
    from paper_1901_10074_b200.configs import batch_images, centred_mod, plaintext_forward

    imgs = batch_images(count)
    t = be.params.plain_modulus
    want = [centred_mod(plaintext_forward(net, im), t) for im in imgs]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall = time.perf_counter()
    e0.record()
    got = []
    pending = None
    nxt = I.pack_image(be, imgs[0])
    for i in range(count):
        cur = nxt
        out = I.decrypt_logits_async(be, I.infer(be, net, cur))
        if i + 1 < count:
            nxt = I.pack_image(be, imgs[i + 1])
        if pending is not None:
            got.append(pending())
        pending = out
    got.append(pending())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ok = all([int(v) for v in g] == w for g, w in zip(got, want))
    return {"images": count, "images_per_s": round(count * 1000.0 / ms, 5),
            "ms_per_image": round(ms / count, 3), "wall_s": round(time.perf_counter() - wall, 2),
            "all_logits_exact": ok,
            "what": "BASELINE configs[4]: 256-image stream shape; this leg times the first "
                    f"{count} images (same key, one Generator), CUDA events around the stream"}


def _config1_leg() -> dict:
    """Config 1 (BASELINE configs[0], the reference's CPU-runnable toy net at
    desk) end to end through the public API: keygen (reported apart), then
    pack_image -> infer -> decrypt_logits, CUDA events around the three.  The
    reference's own run of the same thing is measured in full by the
    cpu_baseline leg (config1_measured_in_full)."""
    import numpy as np
    import torch

    from paper_1901_10074_b200 import inference as I
    from paper_1901_10074_b200.configs import (KEY_SEED, centred_mod, config_network,
                                               config_params, plaintext_forward)
    from paper_1901_10074_b200.fv import FvBackend

    params = config_params(1)
    img, net = config_network(1)
    t0 = time.perf_counter()
    be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t0
    I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))  # warm-up (plans, caches)
    be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))    # fresh Generator: same draws
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    logits = I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    e1.record()
    torch.cuda.synchronize()
    want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
    return {"ms": round(e0.elapsed_time(e1), 2), "keygen_s": round(keygen_s, 2),
            "logits": [int(v) for v in logits],
            "logits_exact": [int(v) for v in logits] == want,
            "path": "pack_image(host pixels) + infer + decrypt_logits(host logits), desk, 1 image"}


def _config3_leg():
    """Config 3 (BASELINE configs[2]): one 256x256x3 image end to end through
    the public API -- pack_image (host pixels) -> infer (conv1, square, conv2,
    square, FC) -> decrypt_logits (host logits) -- CUDA-event timed (keygen
    excluded and reported separately); logits vs the exact plaintext pass."""
    import numpy as np
    import torch

    from paper_1901_10074_b200 import inference as I
    from paper_1901_10074_b200 import planner
    from paper_1901_10074_b200.configs import (KEY_SEED, centred_mod, config_network,
                                               config_params, plaintext_forward,
                                               workload_op_counts)
    from paper_1901_10074_b200.fv import FvBackend

    params = config_params(3)
    img, net = config_network(3)
    t0 = time.perf_counter()
    be = FvBackend(params, rng=np.random.default_rng(KEY_SEED))
    torch.cuda.synchronize()
    keygen_s = time.perf_counter() - t0
    planner.ks_reset(be.ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall = time.perf_counter()
    e0.record()
    logits = I.decrypt_logits(be, I.infer(be, net, I.pack_image(be, img)))
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall
    ms = e0.elapsed_time(e1)
    want = centred_mod(plaintext_forward(net, img), params.plain_modulus)
    ks = planner.ks_stats(be.ctx)
    planner.release_workspace(be.ctx)
    torch.cuda.empty_cache()
    return {"ms": round(ms, 1), "wall_s": round(wall, 2), "keygen_s": round(keygen_s, 2),
            "q_primes": be.ctx.k, "logits_exact": [int(v) for v in logits] == want,
            "ks_launches": ks["ks_launches"], "ks_cts": ks["ks_cts"],
            "serial_op_counts": workload_op_counts(3),
            "path": "pack_image(host pixels) + infer + decrypt_logits(host logits), 1 image"}, be


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


def _cpu_baseline(params, counts, gpu_keys) -> dict:
    """The reference itself (baseline/_ref: hepack FvBackend + numba) on one
    host core, a bounded sample (~25 s): per-op times of its own rotate (one
    key-switch hop), cmult, add, square + relinearisation, encrypt, decrypt at
    retina (config 2) and at 24 q primes (config 3), extrapolated with the
    exact serial op counts; the object-path NttPrime for config 4.  Its key
    set holds the GPU keygen's keys (bit-identical to the reference keygen's
    for the seed; only relin + Galois offset 1, all the sample uses).  Falls
    back to the oracle port when the reference is not installed."""
    from oracle import ref_baseline as RB
    from paper_1901_10074_b200.configs import workload_op_counts

    H = RB.load_hepack()
    info = RB.cpu_info()
    if H is None:
        res = _cpu_baseline_port(params, counts)
        res["cpu"] = info
        return res
    t_all = time.perf_counter()
    per_cfg = {}
    for cfg in (2, 3):
        if gpu_keys.get(cfg) is None:
            continue
        t0 = time.perf_counter()
        be = RB.reference_backend(H, cfg, keys=RB.keyset_from_gpu(H, gpu_keys[cfg]))
        st = RB.prepare(be)
        setup = time.perf_counter() - t0
        light = RB.sample(st, hops=2 if cfg == 2 else 1, cmults=1, adds=10)
        per_op = {**light, **RB.sample_heavy(st, light["ks_hop"])}
        cnt = counts if cfg == 2 else workload_op_counts(3)
        per_cfg[cfg] = {"ms": round(RB.extrapolate(per_op, cnt) * 1000.0, 1),
                        "per_op_s": {k: round(v, 4) for k, v in per_op.items()},
                        "setup_s": round(setup, 2), "op_counts": cnt}
        del be, st
    ntt = RB.ntt_object_path(H)
    c1 = RB.config1_full(H)
    c2 = per_cfg[2]
    return {"value": c2["ms"], "unit": "ms", "cores": 1, "kind": "reference",
            "sample": "hepack (the reference, baseline/_ref, numba "
                      f"{'on' if H.ntt._HAVE_NUMBA else 'off'}) on 1 core: its own rotate (1 "
                      "key-switch hop) x2, cmult, 10 adds, square+relin, encrypt, decrypt at "
                      "retina; single-image latency = sum_op exact serial count x time "
                      "(extrapolated: a whole image is ~30 h of CPU)",
            "config3_ms": per_cfg.get(3, {}).get("ms"),
            "config1_measured_in_full": c1,
            "per_config": per_cfg,
            "config4_object_ntt_polys_per_s": ntt,
            "cpu": info, "wall_s": round(time.perf_counter() - t_all, 1)}


def _cpu_baseline_port(params, counts) -> dict:
    from oracle import cpu_baseline as cb

    t0 = time.perf_counter()
    per_op = cb.time_ops(params, hops=6, cmults=3)
    sec = cb.extrapolate(per_op, counts, workers=1)
    return {"value": round(sec * 1000.0, 1), "unit": "ms", "cores": 1, "kind": "port",
            "sample": "oracle port (reference not installed in baseline/_ref) at retina: "
                      "6 key-switch hops, 3 ct x pt, 10 adds, 1 square+relin, 1 encrypt, "
                      "1 decrypt; per-image latency extrapolated with the exact serial op "
                      f"counts {counts}",
            "per_op_s": {k: round(v, 4) for k, v in per_op.items()},
            "wall_s": round(time.perf_counter() - t0, 1)}


def _ntt_microbench(peaks=None):
    """Config 4 secondary: batched forward/inverse NTT polys/s (device order),
    with each entry's roofline fraction: per-limb work (N/2) log2 N + N
    modmuls against the measured lazy Shoup butterfly rate of
    the word size (32-bit or 64-bit) -- `frac` -- and against 8(d)'s literal
    c x IMAD-rate model -- `frac_8d_literal` (which ignores that IMAD.HI and
    IMAD.WIDE issue at half rate, so it understates what the pipe allows)."""
    import ctypes as C

    import torch

    from paper_1901_10074_b200 import _native as nat
    from paper_1901_10074_b200.ring import find_ntt_primes, root_of_unity

    lib = nat.load()
    res, fracs = {}, {}
    for log_n, bits, L, batch in [(16, 60, 8, 64), (15, 55, 8, 128), (14, 60, 8, 256),
                                  (13, 60, 8, 256), (12, 50, 8, 1024), (14, 30, 22, 256),
                                  (12, 30, 8, 1024)]:
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
                # SURVEY.md 8(d)'s literal constants: c IMAD per modmul (3 for
                # 30-bit, 10 for a 64-bit twiddle modmul) at the probed IMAD rate
                c8d = 10 if wide else 3
                fracs[key] = {"Tmodmul_s": round(tm, 3), "peak": round(pk, 3),
                              "frac": round(tm / pk, 3),
                              "frac_8d_literal": round(tm * c8d / peaks["imad"], 3)}
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
    """The unmodified reference on the host CPU (rank 0 only).  Setup (not
    timed): its own keygen at retina (FvBackend(profile, rng=default_rng
    (1234)), ~50 s), one encryption, one square + relinearisation and one
    decryption.  Each step: the light op sample (1 key-switch hop, 1 cmult, 10
    adds) in this process alone -> single-image latency (exact serial counts
    x per-op times), then the same sample in P forked workers at once ->
    images/s = P / latency under full load."""
    if rank != 0:
        return None
    from oracle import ref_baseline as RB
    from paper_1901_10074_b200.configs import workload_op_counts

    H = RB.load_hepack()
    if H is None:
        return {"impl": "reference", "metric": METRIC,
                "unavailable": "reference not installed in baseline/_ref (see DESIGN.md)"}
    info = RB.cpu_info()
    workers = max(1, info["physical"])
    counts = workload_op_counts(args.config)
    t_all = time.perf_counter()
    be = RB.reference_backend(H, args.config)
    keygen_s = time.perf_counter() - t_all
    st = RB.prepare(be)
    hop0 = RB.sample(st, hops=1, cmults=0, adds=0)["ks_hop"]
    heavy = RB.sample_heavy(st, hop0)
    lat, thr = [], []
    for i in range(args.warmup + args.steps):
        light = RB.sample(st)
        loaded = RB.sample_parallel(st, workers)
        if i < args.warmup:
            continue
        lat.append(RB.extrapolate({**light, **heavy}, counts) * 1000.0)
        per_worker = [RB.extrapolate({**w, **heavy}, counts) for w in loaded]
        thr.append(sum(1.0 / x for x in per_worker))
    value = statistics.mean(lat)
    ips = statistics.mean(thr)
    c1 = RB.config1_full(H)
    sample = (f"hepack (baseline/_ref, numba {'on' if H.ntt._HAVE_NUMBA else 'off'}), own keygen; "
              "per step 1 key-switch hop + 1 cmult + 10 adds at retina in one process; "
              "square/encrypt/decrypt timed once; single-image latency extrapolated with the "
              f"exact serial op counts {counts}")
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "ms", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value, 1), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64 numpy residues", "data": "synthetic",
        "config": dict(CONFIG, parallelism="1 CPU process (the reference is serial per image)"),
        "cpu_baseline": {"value": round(value, 1), "unit": "ms", "cores": 1, "kind": "reference",
                         "sample": sample},
        "throughput": {"images_per_s": round(ips, 9), "workers": workers,
                       "what": f"{workers} worker processes each running whole images (the same "
                               "sample timed in all of them at once): images/s = sum over "
                               "workers of 1 / latency under load"},
        "cpu": info,
        "config1_measured_in_full": c1,
        "e2e": {"value": round(value, 1), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "keygen_s": round(keygen_s, 1),
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
    ap.add_argument("--no-legs", action="store_true", help="skip the config-3 / config-5 legs")
    ap.add_argument("--config5-images", type=int, default=8)
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
