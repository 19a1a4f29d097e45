"""Batched layer planner: the reference's row loop (inference.py:277-349)
re-orchestrated for the GPU, with bit-identical results.

The reference evaluates one weight row at a time: segment ct x pt products
summed, an AllSum fold over s slots (log2 s rotations), an optional bias, a
one-hot mask, a placement rotation by -off, and an add into the output
ciphertext.  Rows are independent until that final modular sum, so the
planner evaluates a tile of T rows per kernel launch:

  1. plaintexts: the tile's sparse segment vectors are encoded on the device
     (sparse scatter + inverse t-NTT), centred, reduced to every q prime and
     transformed (hefv_encode_sparse, hefv_plain_to_rns);
  2. segment products: one launch multiplies them against the NTTs of the
     layer's input ciphertexts and sums per row in the NTT domain
     (hefv_rows_mac) -- equal to the reference's cmult + add chain because
     the NTT is linear and modular addition is order-free;
  3. AllSum step j (shift 2^j) for all rows of the tile: one automorphism
     launch + one fused key-switch launch under the shared Galois key, with
     the running-sum addition fused into the key-switch epilogue;
  4. biases (batched add_plain), the e0 mask (batched ct x pt);
  5. placement: rotation by -off decomposes into ascending power-of-two hops
     (fv.py:422-425); hop 2^b for every row whose offset has bit b set is one
     batched launch, bits ascending, so each row sees its hops in the
     reference's order;
  6. per-output-ciphertext modular sums of the pieces (hefv_accumulate_rows).

Steps 1-6 run in C++ (hefv_layer_rows, csrc/layer.cu) from one call per
layer: this module builds the host plan (CSR plaintexts, per-row output /
offset / bias), sizes the workspaces, checks depths and replays the ledger.

Every ciphertext the planner produces has exactly the limbs the serial
schedule produces (the key-switch noise depends only on the ciphertext being
switched, which is the same), the Generator is consumed exactly as in the
reference (only the final bias-only encryptions draw), and the CostReport
ledger is replayed from a host simulation of the serial schedule.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .errors import DepthBudgetError

_TILE_BYTES = 24 << 30  # device memory budget for one tile's working set


def keyswitch_call(ctx, key, *args, dig_slot=None, galois=0):
    """One batched key switch under ``key`` (a SwitchKey); ``args`` are
    hefv_keyswitch's after the key pointers (the batch size last).  Keys with
    an aux-basis form go through hefv_keyswitch_aux (same limbs, fewer
    transforms), which can also read the digit rows through a slot map and
    apply a Galois automorphism on the fly (``dig_slot`` device pointer,
    ``galois`` element); the per-prime kernel needs its digits materialised.
    Calls and ciphertexts are counted by the library (``ks_stats``)."""
    batch = int(args[-1])
    if key.aux_dev is not None:
        scratch, cap = _ks_workspace(ctx, batch)
        ctx.call("hefv_keyswitch_aux", key.aux_dev.data_ptr(), args[0], args[1], dig_slot,
                 int(galois), *args[2:-1], scratch.data_ptr(), cap, batch, ctx.stream())
    else:
        if dig_slot is not None or galois:
            raise ValueError("the per-prime key switch needs materialised digits")
        ctx.call("hefv_keyswitch", key.body_dev.data_ptr(), key.mask_dev.data_ptr(), *args,
                 ctx.stream())


def ks_reset(ctx, timing: bool = False) -> None:
    """Zero the library's key-switch counters of ``ctx``; with ``timing`` a
    CUDA event pair brackets every later key-switch call (hefv_ks_timing)."""
    ctx.call("hefv_ks_timing", 1 if timing else 0)


def ks_stats(ctx) -> dict:
    """Key-switch calls, ciphertexts and (with timing on) summed device ms
    since the last ``ks_reset`` (hefv_ks_stats; synchronises on the events)."""
    import ctypes as C

    calls, cts, ms = C.c_int64(), C.c_int64(), C.c_double()
    ctx.call("hefv_ks_stats", C.byref(calls), C.byref(cts), C.byref(ms))
    return {"ks_launches": calls.value, "ks_cts": cts.value, "ks_ms": ms.value}


def rotation_keyswitch(ctx, key, src, src_stride, slot, g, B, out0, out1, out_stride, out_slot,
                       adB0, adB1, adB_stride, scratch):
    """One Galois hop of B ciphertexts (fv.py:417-432, 157-173):
    out[out_slot b] = KS(sigma_g(c1)) + (sigma_g(c0), 0) + adB[out_slot b]
    with c = the ciphertext at src + slot[b] * src_stride (words; slot may be
    None).  With an aux-basis key only sigma_g(c0) is materialised (into
    ``scratch``, >= B k N words) and sigma_g(c1) is applied inside the key
    switch's digit load; otherwise both parts go through ``scratch`` (>= 2 B
    k N words)."""
    stack = ctx.k * ctx.n
    st = ctx.stream()
    if key.aux_dev is not None:
        ctx.call("hefv_automorph", src, src_stride, slot, scratch, 1, g, B, st)
        keyswitch_call(ctx, key, src + stack * 4, src_stride, out0, out1, out_stride, out_slot,
                       scratch, None, stack, adB0, adB1, adB_stride, B, dig_slot=slot, galois=g)
    else:
        ctx.call("hefv_automorph", src, src_stride, slot, scratch, 2, g, B, st)
        keyswitch_call(ctx, key, scratch + stack * 4, 2 * stack, out0, out1, out_stride, out_slot,
                       scratch, None, 2 * stack, adB0, adB1, adB_stride, B)


KS_WORKSPACE_BYTES = 24 << 30  # ~1900 ciphertexts per chunk at retina: one chunk per config-2 launch
MEM_FRACTION = 0.3              # of the free device memory, per budget (workspace, tile)


def _budget(limit: int, held: int = 0) -> int:
    """``limit`` clamped to MEM_FRACTION of the device memory free now (plus
    what the caller already holds and would give back)."""
    import torch

    free, _ = torch.cuda.mem_get_info()
    return int(min(limit, MEM_FRACTION * (free + held)))


def _ks_workspace(ctx, batch: int):
    """Scratch of the aux-basis key switch (9 k N words per ciphertext),
    cached on the context per CUDA stream (work queued on two streams must
    not share it; ``release_workspace`` drops them); ciphertexts beyond its
    capacity run in chunks.  Sized from KS_WORKSPACE_BYTES and the free
    device memory, so several live contexts do not each pin 24 GB."""
    import torch

    per_ct = 9 * ctx.k * ctx.n
    cache = getattr(ctx, "_ks_ws", None)
    if cache is None:
        cache = ctx._ks_ws = {}
    key = torch.cuda.current_stream().cuda_stream
    ws = cache.get(key)
    held = 0 if ws is None else ws.numel() * 4
    if ws is not None and ws.numel() >= min(batch, KS_WORKSPACE_BYTES // (4 * per_ct)) * per_ct:
        return ws, ws.numel() // per_ct
    cap = max(1, min(batch, _budget(KS_WORKSPACE_BYTES, held) // (4 * per_ct)))
    if ws is None or ws.numel() < cap * per_ct:
        cache[key] = ws = None      # the old buffer is freed before the new one is allocated
        cache[key] = ws = torch.empty(cap * per_ct, dtype=torch.int32, device="cuda")
    return ws, ws.numel() // per_ct


def release_workspace(ctx) -> None:
    """Drop the key-switch workspaces cached on ``ctx``."""
    ctx._ks_ws = None


def count_layer_ops(rows, x_k: int, s: int, slot_count: int, galois_offsets,
                    skip_zero_segments=True) -> dict:
    """Exact op counts of the serial schedule for one compiled layer
    (inference.py:277-349), plus the key-switch hops its rotations cost."""
    n_iter = _allsum_iters(s)
    tot = {"cmult": 0, "add": 0, "rotation": 0, "encrypt": 0, "ks_hops": 0}
    seen, biased_only = set(), set()
    for r in rows:
        nseg = len(r.segment_ids) if skip_zero_segments else x_k
        m, off = divmod(r.out_index, s)
        if nseg == 0:
            if r.bias:
                biased_only.add(m)
            continue
        counts, _, _ = _row_events(nseg, n_iter, bool(r.bias), bool(off), m not in seen)
        seen.add(m)
        for f, v in counts.items():
            tot[f] += v
        tot["ks_hops"] += n_iter
        if off:
            rot = (-off) % slot_count
            tot["ks_hops"] += 1 if rot in galois_offsets else bin(rot).count("1")
    nout = max(1, -(-len(rows) // s))
    for m in range(nout):
        if m not in seen:
            tot["encrypt"] += 1
        elif m in biased_only:
            tot["add"] += 1
    return tot


# ---------------------------------------------------------------------------
# ledger replay of the serial schedule
# ---------------------------------------------------------------------------
_EVENT_CACHE: dict = {}


def _row_events(nseg: int, n_iter: int, has_bias: bool, has_off: bool, first: bool):
    """Counts, net live change and peak (relative) of one row of the serial
    schedule (inference.py:302-338 + engine.py:309-327)."""
    key = (nseg, n_iter, has_bias, has_off, first)
    hit = _EVENT_CACHE.get(key)
    if hit is not None:
        return hit
    counts = {"cmult": 0, "add": 0, "rotation": 0}
    live = peak = 0

    def new(field):
        nonlocal live, peak
        counts[field] += 1
        live += 1
        peak = max(peak, live)

    def drop(c=1):
        nonlocal live
        live -= c

    for i in range(nseg):
        new("cmult")
        if i:
            new("add")
            drop(2)
    for i in range(n_iter):  # all_sum
        new("rotation")
        new("add")
        drop(1)  # release(r)
        if i:
            drop(1)  # release(cur) when cur is not the input
    if n_iter:
        drop(1)  # dot is not acc: release(acc)
    if has_bias:
        new("add")
        drop(1)
    new("cmult")  # piece = cmult(dot, e0)
    drop(1)       # release(dot)
    if has_off:
        new("rotation")
        drop(1)
    if not first:
        new("add")
        drop(2)
    res = (counts, live, peak)
    _EVENT_CACHE[key] = res
    return res


# ---------------------------------------------------------------------------
# the planner
# ---------------------------------------------------------------------------
def replay_ledger(ledger, rows, x_k, s, width, n_iter, m_arr, off_arr, bias_arr, nseg,
                  row_level):
    """Apply the serial schedule's ledger events for a layer, in row order.
    Returns (output ciphertexts that receive pieces, bias-only plaintexts)."""
    seen_m = set()
    plain_bias = {}
    for i in range(len(rows)):
        m = int(m_arr[i])
        if not nseg[i]:
            if bias_arr[i]:
                plain_bias.setdefault(m, np.zeros(width, dtype=np.int64))[int(off_arr[i])] += bias_arr[i]
            continue
        first = m not in seen_m
        seen_m.add(m)
        counts, dlive, peak = _row_events(int(nseg[i]), n_iter, bool(bias_arr[i]),
                                          bool(off_arr[i]), first)
        ledger.absorb(counts, dlive, peak, int(row_level[i]) + 1)
    return seen_m, plain_bias


def _allsum_iters(s: int) -> int:
    n, shift = 0, 1
    while shift < s:
        n += 1
        shift <<= 1
    return n


def planned_layer_eval(backend, rows, x, skip_zero_segments=True, scale_factor=1):
    import torch

    from .inference import PackedVector

    ctx = backend.ctx
    params = backend.params
    s = x.slots_used
    width = params.slot_count
    t = params.plain_modulus
    kq, n = ctx.k, ctx.n
    R = len(rows)
    nout = max(1, -(-R // s))
    n_iter = _allsum_iters(s)
    x_levels = [ct.level_used for ct in x.cts]

    # ---- host plan ------------------------------------------------------------
    out_index = np.fromiter((r.out_index for r in rows), dtype=np.int64, count=R)
    m_arr = out_index // s
    off_arr = out_index % s
    bias_arr = [int(r.bias) for r in rows]
    seg_lists = [r.segment_ids if skip_zero_segments else np.arange(x.k) for r in rows]
    nseg = np.fromiter((len(sl) for sl in seg_lists), dtype=np.int64, count=R)
    has_acc = nseg > 0
    # depth checks up front (the serial schedule raises at the first offending cmult)
    budget = params.depth_budget
    row_level = np.zeros(R, dtype=np.int64)
    act = np.nonzero(has_acc)[0]
    if len(act):
        segs = np.concatenate([np.asarray(seg_lists[i], dtype=np.int64) for i in act])
        starts = np.concatenate(([0], np.cumsum(nseg[act])[:-1]))
        lv = np.maximum.reduceat(np.asarray(x_levels, dtype=np.int64)[segs], starts) + 1
        over = np.nonzero(lv + 1 > budget)[0]  # the cmult (lv) or the e0 mask (lv + 1)
        if len(over):
            first = int(lv[over[0]])
            bad = first if first > budget else first + 1
            raise DepthBudgetError(f"operation needs level {bad} but depth_budget is {budget}")
        row_level[act] = lv

    # ---- device work (queued chunk by chunk; the host plans chunk c + 1 while
    # the GPU runs chunk c) -----------------------------------------------------------
    active = act
    out_dev = torch.zeros((nout, 2, kq, n), dtype=torch.int32, device="cuda")
    out_level_arr = np.zeros(nout, dtype=np.int64)
    np.maximum.at(out_level_arr, m_arr[active], row_level[active] + 1)
    out_level = [int(v) for v in out_level_arr]
    if len(active):
        _run_rows(backend, rows, x, seg_lists, active, m_arr, off_arr, bias_arr, out_dev,
                  n_iter, skip_zero_segments)

    # the ledger of the serial schedule (host accounting; the device work does
    # not touch it, so replaying it after the launches keeps the event order)
    seen_m, plain_bias = replay_ledger(backend._c, rows, x_k=x.k, s=s, width=width,
                                       n_iter=n_iter, m_arr=m_arr, off_arr=off_arr,
                                       bias_arr=bias_arr, nseg=nseg, row_level=row_level)

    # ---- outputs + the reference's final loop (inference.py:342-348) ----------
    from .fv import FvCiphertext

    out = []
    for m in range(nout):
        if m in seen_m:
            out.append(FvCiphertext(None, out_level[m], params, dev=out_dev[m]))
        else:
            out.append(None)
    for m in range(nout):
        if out[m] is None:
            out[m] = backend.encrypt(plain_bias.get(m, np.zeros(width, dtype=np.int64)))
        elif m in plain_bias:
            nxt = backend.add_plain(out[m], plain_bias[m])
            backend.release(out[m])
            out[m] = nxt
    del t
    return PackedVector(R, s, out, scale=x.scale * scale_factor)


def _sparse_plan(rows, order, s: int, t: int) -> dict:
    """CSR of every (row, nonzero segment) plaintext, rows in `order`:
    entries (slot, value mod t) grouped by plaintext, plaintexts grouped by
    row (row_ptr), each tagged with its input segment.  Vectorised over the
    whole layer -- identical to segment_dense (inference.py:68-73) per row."""
    lens = np.fromiter((len(rows[i].positions) for i in order), dtype=np.int64, count=len(order))
    if lens.sum() == 0:
        z = np.zeros(1, dtype=np.int64)
        return {"ptr": z, "slot": np.zeros(0, np.int32), "val": np.zeros(0, np.uint64),
                "row_ptr": np.zeros(len(order) + 1, dtype=np.int64), "seg": np.zeros(0, np.int32)}
    pos = np.concatenate([np.asarray(rows[i].positions, dtype=np.int64) for i in order])
    raw = [np.asarray(rows[i].values) for i in order]
    if any(v.dtype == object for v in raw):
        val = np.array([int(w) % t for v in raw for w in v], dtype=np.uint64)
    else:
        val = np.mod(np.concatenate(raw).astype(np.int64), t).astype(np.uint64)
    ridx = np.repeat(np.arange(len(order), dtype=np.int64), lens)
    seg = pos // s
    # group by (row, segment), position order kept inside a segment; compiled
    # conv / fc rows list their positions ascending, so this is usually the
    # identity and the sort is skipped
    if len(seg) > 1 and not np.all((ridx[1:] > ridx[:-1]) | (seg[1:] >= seg[:-1])):
        perm = np.lexsort((seg, ridx))  # stable
        pos, val, ridx, seg = pos[perm], val[perm], ridx[perm], seg[perm]
    key = ridx * (int(seg.max()) + 1) + seg
    starts = np.flatnonzero(np.concatenate(([True], key[1:] != key[:-1])))
    ptr = np.concatenate((starts, [len(key)])).astype(np.int64)
    g_row = ridx[starts]
    row_ptr = np.searchsorted(g_row, np.arange(len(order) + 1), side="left").astype(np.int64)
    return {"ptr": ptr, "slot": (pos % s).astype(np.int32), "val": val, "row_ptr": row_ptr,
            "seg": seg[starts].astype(np.int32)}


def _tile_rows(backend, n_plain_per_row: float) -> int:
    ctx = backend.ctx
    ct_bytes = 2 * ctx.k * ctx.n * 4
    per_row = 2 * ct_bytes + n_plain_per_row * (ctx.k * ctx.n * 4 + ctx.n * 8)
    # a tile's (T, 2, k, N) word count stays below 2^31 (32-bit element indices)
    words_cap = ((1 << 31) - 1) // (2 * ctx.k * ctx.n)
    return int(max(1, min(8192, words_cap, _budget(_TILE_BYTES) // per_row)))


def _run_rows(backend, rows, x, seg_lists, active, m_arr, off_arr, bias_arr, out_dev, n_iter,
              skip_zero_segments):
    """The device work of a layer: hefv_layer_rows calls (layer.cu) over the
    active rows, grouped by output ciphertext, in chunks so that the host
    plans chunk c + 1 while the GPU runs chunk c.  Python only builds the
    host plan (CSR plaintexts, per-row output / offset / bias) and the
    workspaces; tiling, AllSum, biases, the e0 mask, placement hops and the
    output sums run in C++."""
    import torch

    ctx = backend.ctx
    s = x.slots_used
    xin = torch.stack([backend.dev(ct)[:2] for ct in x.cts]).contiguous()
    order = active[np.argsort(m_arr[active], kind="stable")]
    avg_plain = max(1.0, float(np.mean([len(seg_lists[i]) for i in order])))
    T = _tile_rows(backend, avg_plain)
    # one tile first (its planning is the only host time the GPU waits for),
    # then growing chunks planned while the previous ones run
    lo, size = 0, T
    while lo < len(order):
        _layer_rows_call(backend, rows, xin, len(x.cts), order[lo:lo + size], m_arr, off_arr,
                         bias_arr, out_dev, n_iter, s, T)
        lo += size
        size = min(8 * T, 2 * size)


def _layer_rows_call(backend, rows, xin, x_cts, order, m_arr, off_arr, bias_arr, out_dev, n_iter,
                     s, T):
    """One hefv_layer_rows call over the rows ``order`` (grouped by output)."""
    import ctypes as C

    import torch

    ctx = backend.ctx
    t = backend.params.plain_modulus
    R = len(order)
    plan = _sparse_plan(rows, order, s, t)
    row_out = np.ascontiguousarray(m_arr[order], dtype=np.int32)
    row_off = np.ascontiguousarray(off_arr[order], dtype=np.int32)
    row_bias = np.array([int(bias_arr[i]) % t for i in order], dtype=np.uint64)
    row_ptr = np.ascontiguousarray(plan["row_ptr"], dtype=np.int64)
    plain_ptr = np.ascontiguousarray(plan["ptr"], dtype=np.int64)
    plain_seg = np.ascontiguousarray(plan["seg"], dtype=np.int32)
    slot_idx = np.ascontiguousarray(plan["slot"], dtype=np.int32)
    slot_val = np.ascontiguousarray(plan["val"], dtype=np.uint64)
    galois = backend.keys.galois
    offsets = np.array(sorted(galois), dtype=np.int32)
    handles = (C.c_void_p * len(offsets))(*[galois[int(o)].handle.value for o in offsets])

    def ptr(a):
        return a.ctypes.data if a.size else None

    words = C.c_int64()
    ctx.call("hefv_layer_rows_work_words", x_cts, R, ptr(row_ptr), T, C.byref(words))
    work = torch.empty(words.value, dtype=torch.int32, device="cuda")
    if ctx.ks_aux:
        ws, cap = _ks_workspace(ctx, T)
        ws_ptr = ws.data_ptr()
    else:
        ws_ptr, cap = None, 0
    h2d0 = C.c_int64()
    ctx.call("hefv_transfer_stats", C.byref(h2d0), None)
    ctx.call("hefv_layer_rows", xin.data_ptr(), x_cts, R, ptr(row_out), ptr(row_off),
             ptr(row_bias), ptr(row_ptr), ptr(plain_seg), ptr(plain_ptr), ptr(slot_idx),
             ptr(slot_val), n_iter, backend.params.slot_count, len(offsets), ptr(offsets),
             handles, out_dev.data_ptr(), out_dev.shape[0], T, work.data_ptr(), words.value,
             ws_ptr, cap, ctx.stream())
    h2d1 = C.c_int64()
    ctx.call("hefv_transfer_stats", C.byref(h2d1), None)
    nat.TRAFFIC["h2d"] += h2d1.value - h2d0.value   # the plan, staged and copied by the library
