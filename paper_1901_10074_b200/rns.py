"""Standalone RNS key switch over 64-bit primes (BASELINE config 4).

Config 4 asks for a full key switch with L in {1, 2, 4, 8} NTT-friendly
primes of 50-60 bits (p = 1 mod 2N), N in 2^12..2^16 -- the reference's
`_keyswitch_apply` (fv.py:205-217) run over `_FvContext(FvParams(n, t,
q_primes))` with such primes (its object-dtype path).  `RnsKeySwitch64`
holds the device tables for that prime set and runs the switch on the GPU
(`hefv_keyswitch64`).  Keys are taken in the reference's layout
(`SwitchKey.body[j]` = (L digits, N) natural-order NTT stacks) and stored in
device order, Montgomery form.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .ring import bitrev_perm, root_of_unity


class RnsKeySwitch64:
    def __init__(self, primes, n: int):
        import torch

        nat.require_device()
        lib = nat.load()
        self.primes = [int(p) for p in primes]
        self.L = len(self.primes)
        self.n = n
        self.log_n = n.bit_length() - 1
        if any(p >= 1 << 62 for p in self.primes):
            raise ValueError("primes must be below 2^62")
        psis = [root_of_unity(p, n) for p in self.primes]
        h = C.c_void_p()
        nat.check(lib.hefv_ctx_create(C.byref(h), self.log_n, 0, None, None, self.L,
                                      (C.c_uint64 * self.L)(*self.primes),
                                      (C.c_uint64 * self.L)(*psis)), "hefv_ctx_create")
        self._h = h
        self._torch = torch
        self.brev = bitrev_perm(self.log_n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and nat._lib is not None:
            nat._lib.hefv_ctx_destroy(h)
            self._h = None

    def _dev(self, arr):
        return nat.to_device(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64)).view(np.int64))

    def upload_key(self, body, mask):
        """body/mask: lists over target prime j of (L, N) natural-order residues."""
        out = []
        for part in (body, mask):
            stack = np.stack([np.asarray(part[j], dtype=object) for j in range(self.L)])
            dev_order = stack[..., self.brev].astype(np.uint64)
            t = self._dev(dev_order.reshape(-1, self.L, self.n))  # rows = L (digits)...
            # rows: (j, i) -> prime j; Montgomery conversion wants prime = row % L over
            # (rows, L, N) -- transpose so the prime index is the middle axis
            t = t.view(self.L, self.L, self.n).transpose(0, 1).contiguous()  # [i][j]
            m = self._torch.empty_like(t)
            nat.call("hefv_to_montgomery64", self._h, t.data_ptr(), m.data_ptr(), self.L,
                     nat.stream_handle())
            out.append(m.transpose(0, 1).contiguous())  # back to [j][i]
        return tuple(out)

    def random_key(self, seed: int = 0):
        """Uniform key material (timing only)."""
        torch = self._torch
        g = torch.Generator(device="cuda").manual_seed(seed)
        p = torch.tensor(self.primes, dtype=torch.int64, device="cuda").view(self.L, 1, 1)
        mk = lambda: torch.randint(0, 1 << 62, (self.L, self.L, self.n), dtype=torch.int64,  # noqa: E731
                                   device="cuda", generator=g) % p
        return mk(), mk()

    def switch(self, key, digits_dev):
        """digits_dev: (B, L, N) int64 residues; returns (B, 2, L, N) coefficients."""
        torch = self._torch
        B = digits_dev.shape[0]
        out = torch.empty((B, 2, self.L, self.n), dtype=torch.int64, device="cuda")
        scratch = torch.empty((B, self.L, self.L, self.n), dtype=torch.int64, device="cuda")
        nat.call("hefv_keyswitch64", self._h, key[0].data_ptr(), key[1].data_ptr(),
                 digits_dev.data_ptr(), out.data_ptr(), scratch.data_ptr(), B,
                 nat.stream_handle())
        return out

    def switch_host(self, key, digits):
        d = self._dev(np.asarray(digits, dtype=object).astype(np.uint64))
        return nat.to_host(self.switch(key, d.view(-1, self.L, self.n))).astype(object)
