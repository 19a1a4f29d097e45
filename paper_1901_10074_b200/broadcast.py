"""Batched interleaved (per-pixel broadcast) layers on the GPU backend.

The reference's CryptoNets-style baseline (inference.py:379-438) keeps one
ciphertext per neuron with the value broadcast to every slot; a linear layer
is, per output row, a chain of ``cmult(vals[pos], np.full(width, w))`` and
``add``, an ``add_plain`` of the broadcast bias, or an ``encrypt`` of the bias
when the row has no taps.

Every cmult by the broadcast weight w uses the same plaintext
centred(encode(full(w))) (the encoding fills only the N/2 batching slots, so
it is a full polynomial, not a constant), so the layer needs one plaintext
NTT per distinct weight value and one NTT of every input ciphertext; each
row's cmult + add chain is then a single NTT-domain sum followed by one
inverse NTT (hefv_rows_mac_indexed) -- identical limbs, since the NTT is
linear and modular addition is order-free.  Broadcast biases are one
Delta*m plaintext per distinct bias value added to part 0 (hefv_add_part0).
The ledger is replayed from the serial schedule's event sequence, and
bias-only rows are encrypted in row order so the Generator is consumed
exactly as in the reference.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat


def row_events(ntaps: np.ndarray, has_bias: np.ndarray):
    """Ledger effect of the serial row loop (inference.py:406-428): op counts
    and the live-count peak relative to the layer's start (each row leaves
    one ciphertext live; inside a row, acc + product + sum are live at once)."""
    ntaps = np.asarray(ntaps, dtype=np.int64)
    has_bias = np.asarray(has_bias, dtype=bool)
    nonempty = ntaps > 0
    extra = np.where(ntaps >= 2, 3, np.where(nonempty & has_bias, 2, 1))
    peak_rel = int((np.arange(len(ntaps)) + extra).max(initial=0))
    counts = {
        "cmult": int(ntaps.sum()),
        "add": int(np.maximum(ntaps - 1, 0).sum() + (nonempty & has_bias).sum()),
        "encrypt": int((~nonempty).sum()),
    }
    return counts, peak_rel


def broadcast_layer_eval(backend, rows, vals):
    """All rows of an interleaved linear layer in one launch; returns the
    output ciphertext list, or None when a cmult would exceed the depth
    budget (the caller then runs the serial loop, which raises at the same
    point)."""
    from .fv import FvCiphertext

    torch = __import__("torch")
    ctx = backend.ctx
    t = ctx.t
    levels = np.array([ct.level_used for ct in vals], dtype=np.int64)
    ntaps = np.array([len(r.positions) for r in rows], dtype=np.int64)
    srcs = (np.concatenate([np.asarray(r.positions, dtype=np.int64) for r in rows])
            if len(rows) else np.zeros(0, np.int64))
    out_level = np.zeros(len(rows), dtype=np.int64)
    if srcs.size:
        need = levels[srcs] + 1
        if int(need.max()) > backend.params.depth_budget:
            return None
        starts = np.concatenate([[0], np.cumsum(ntaps)[:-1]])
        nz = ntaps > 0
        out_level[nz] = np.maximum.reduceat(need, starts[nz])
    for ct in vals:
        backend._check_params(ct)
    if not rows:
        return []

    width = backend.params.slot_count
    st = ctx.stream()
    biases = [int(r.bias) for r in rows]
    out = torch.empty((len(rows), 2, ctx.k, ctx.n), dtype=torch.int32, device="cuda")
    if srcs.size:
        # one plaintext per distinct weight value (mod t), as _cmult builds it
        wvals = np.concatenate([np.asarray(r.values, dtype=object) for r in rows]) % t
        uniq, tap_plain = np.unique(wvals.astype(np.uint64), return_inverse=True)
        polys = backend._encode_dev(np.repeat(uniq[:, None], width, axis=1))
        m_ntt = backend._rns_plain(polys, 1, True, False)
        del polys
        used = np.unique(srcs)
        remap = np.full(len(vals), -1, dtype=np.int64)
        remap[used] = np.arange(len(used))
        # NTT (Montgomery, device order) of every input that a tap reads, in
        # chunks so the transient copies stay small next to the layer's inputs
        x_ntt = torch.empty((len(used), 2, ctx.k, ctx.n), dtype=torch.int32, device="cuda")
        for lo in range(0, len(used), 256):
            xin = torch.stack([backend.dev(vals[int(i)])[:2] for i in used[lo:lo + 256]])
            x_ntt[lo:lo + 256] = ctx.to_mont(
                ctx.ntt_q(xin.view(-1, ctx.k, ctx.n)).view_as(xin))
            del xin
        row_ptr = np.concatenate([[0], np.cumsum(ntaps)]).astype(np.int32)
        tap_src = remap[srcs].astype(np.int32)
        tap_plain = tap_plain.astype(np.int32)
        for lo in range(0, len(rows), 65535):
            hi = min(len(rows), lo + 65535)
            rp = row_ptr[lo:hi + 1]
            d_rp = nat.to_device(rp - rp[0])
            d_src = nat.to_device(tap_src[rp[0]:rp[-1]])
            d_pl = nat.to_device(tap_plain[rp[0]:rp[-1]])
            ctx.call("hefv_rows_mac_indexed", x_ntt.data_ptr(), m_ntt.data_ptr(),
                     d_rp.data_ptr(), d_src.data_ptr(), d_pl.data_ptr(), out[lo].data_ptr(),
                     hi - lo, st)
        del x_ntt
        # broadcast biases of rows with taps: part 0 += Delta * encode(full(b))
        bias_rows = [i for i, b in enumerate(biases) if b and ntaps[i] > 0]
        if bias_rows:
            bv = np.array([biases[i] % t for i in bias_rows], dtype=object)
            ub, b_inv = np.unique(bv.astype(np.uint64), return_inverse=True)
            dm = backend._delta_m_dev(np.repeat(ub[:, None], width, axis=1))
            add = dm[torch.as_tensor(b_inv, device="cuda")].contiguous()
            slot = nat.to_device(np.array(bias_rows, dtype=np.int32))
            ctx.call("hefv_add_part0", out.data_ptr(), 2 * ctx.k * ctx.n, slot.data_ptr(),
                     add.data_ptr(), len(bias_rows), st)

    res = [FvCiphertext(None, int(out_level[i]), backend.params, dev=out[i])
           for i in range(len(rows))]
    empty = [i for i in range(len(rows)) if ntaps[i] == 0]
    if empty:
        plains = [backend.as_plain(np.full(width, biases[i], dtype=np.int64)) for i in empty]
        for i, ct in zip(empty, backend._encrypt_many(plains)):
            res[i] = ct
    counts, peak_rel = row_events(ntaps, np.array([b != 0 for b in biases]))
    max_level = int(out_level.max(initial=0))
    backend._c.absorb(counts, len(rows), peak_rel, max_level)
    return res


def square_layer(backend, vals, release_inputs=True):
    """Slot-wise squares of a layer's ciphertexts as batched tensor +
    relinearisation launches, limb-identical to ``mult(ct, ct)`` each.

    ``release_inputs``: the interleaved loop ``mult(ct, ct); release(ct)``
    (inference.py:401-405), else the compact ``square_activation``
    (inference.py:352-355), which keeps its inputs.  The ledger is replayed in
    that serial order.  Returns None when a square would exceed the depth
    budget (the caller's serial loop then raises at the same point)."""
    from .fv import FvCiphertext

    for ct in vals:
        backend._check_params(ct)
    levels = [ct.level_used + 1 for ct in vals]
    if not vals:
        return []
    if max(levels) > backend.params.depth_budget:
        return None
    devs = backend._square_many_dev([backend.dev(ct) for ct in vals])
    out = [FvCiphertext(None, lv, backend.params, dev=d) for lv, d in zip(levels, devs)]
    cur = peak = freed = 0
    for ct in vals:
        cur += 1
        peak = max(peak, cur)
        if release_inputs and ct._live:
            ct._live = False
            cur -= 1
            freed += 1
    backend._c.absorb({"mult": len(vals)}, len(vals), peak, max(levels))
    backend._c.drop(freed)
    return out
