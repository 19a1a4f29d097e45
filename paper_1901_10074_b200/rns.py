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
from .ring import bitrev_perm, find_ntt_primes, root_of_unity


class Key64:
    """A switch key on the device: ``mont`` = (body, mask) (L, L, N) [j][i]
    device order, Montgomery form (direct path); ``aux`` = (T, 2L, L, N) u32
    aux-basis form (None without an aux basis)."""

    def __init__(self, mont, aux):
        self.mont = mont
        self.aux = aux

    def __getitem__(self, i):  # legacy (body, mask) tuple access
        return self.mont[i]


def aux_prime_count(primes, log_n: int, a_bits: float = 29.45) -> int:
    """Aux primes (~2^29.45 each) needed for an exact sum_i c_i (*) B_ji:
    prod a_t > 8 L N max(p)^2 (ks64_aux.cu)."""
    need = 3 + (len(primes) - 1).bit_length() + log_n + 2 * max(primes).bit_length()
    return -(-need // int(a_bits))


class RnsKeySwitch64:
    """``aux``: also run the key switch through an auxiliary basis of ~29.5-bit
    NTT primes (hefv_keyswitch64_aux) -- the same limbs as the direct 64-bit
    path (hefv_keyswitch64) with about a third of the transform work but
    more memory traffic.  Default: for 5 <= L <= 8, where it is measured
    faster on a B200 (L = 8: 24.5 -> 16.9 us at N = 2^14; L = 4 equal; L <= 2
    slower)."""

    def __init__(self, primes, n: int, aux=None):
        import torch

        nat.require_device()
        lib = nat.load()
        self.primes = [int(p) for p in primes]
        self.L = len(self.primes)
        self.n = n
        self.log_n = n.bit_length() - 1
        if any(p >= 1 << 62 for p in self.primes):
            raise ValueError("primes must be below 2^62")
        self.aux = (5 <= self.L <= 8 and 10 <= self.log_n <= 16) if aux is None else bool(aux)
        self.aux_primes = []
        if self.aux:
            T = aux_prime_count(self.primes, self.log_n)
            self.aux_primes = find_ntt_primes(T, 30, 2 * n, below=int(2 ** 29.5))
        psis = [root_of_unity(p, n) for p in self.primes]
        apsis = [root_of_unity(p, n) for p in self.aux_primes]
        T = len(self.aux_primes)
        h = C.c_void_p()
        nat.check(lib.hefv_ctx_create(C.byref(h), self.log_n, T,
                                      (C.c_uint32 * T)(*self.aux_primes) if T else None,
                                      (C.c_uint32 * T)(*apsis) if T else None, self.L,
                                      (C.c_uint64 * self.L)(*self.primes),
                                      (C.c_uint64 * self.L)(*psis)), "hefv_ctx_create")
        self._h = h
        if self.aux:
            nat.check(lib.hefv_ks64_aux_setup(h, T), "hefv_ks64_aux_setup")
        self._torch = torch
        self.brev = bitrev_perm(self.log_n)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and nat._lib is not None:
            nat._lib.hefv_ctx_destroy(h)
            self._h = None

    def _dev(self, arr):
        return nat.to_device(np.ascontiguousarray(np.asarray(arr, dtype=np.uint64)).view(np.int64))

    def _make_key(self, body_dev, mask_dev):
        """body/mask: (L, L, N) [j][i] device-order plain residues on the device."""
        mont = []
        for t in (body_dev, mask_dev):
            # Montgomery conversion wants the prime as the middle axis: [i][j]
            tt = t.transpose(0, 1).contiguous()
            m = self._torch.empty_like(tt)
            nat.call("hefv_to_montgomery64", self._h, tt.data_ptr(), m.data_ptr(), self.L,
                     nat.stream_handle())
            mont.append(m.transpose(0, 1).contiguous())  # back to [j][i]
        aux = None
        if self.aux:
            torch = self._torch
            L, n, T = self.L, self.n, len(self.aux_primes)
            aux = torch.empty((T, 2 * L, L, n), dtype=torch.int32, device="cuda")
            scratch = torch.empty(((4 + T) * L * L * n,), dtype=torch.int64, device="cuda")
            b = body_dev.contiguous()
            m = mask_dev.contiguous()
            nat.call("hefv_ks64_aux_key", self._h, b.data_ptr(), m.data_ptr(), aux.data_ptr(),
                     scratch.data_ptr(), nat.stream_handle())
        return Key64(tuple(mont), aux)

    def upload_key(self, body, mask):
        """body/mask: lists over target prime j of (L, N) natural-order residues."""
        dev = []
        for part in (body, mask):
            stack = np.stack([np.asarray(part[j], dtype=object) for j in range(self.L)])
            dev_order = stack[..., self.brev].astype(np.uint64)
            dev.append(self._dev(dev_order).view(self.L, self.L, self.n))
        return self._make_key(*dev)

    def random_key(self, seed: int = 0):
        """Uniform key material (timing only)."""
        torch = self._torch
        g = torch.Generator(device="cuda").manual_seed(seed)
        p = torch.tensor(self.primes, dtype=torch.int64, device="cuda").view(self.L, 1, 1)
        mk = lambda: torch.randint(0, 1 << 62, (self.L, self.L, self.n), dtype=torch.int64,  # noqa: E731
                                   device="cuda", generator=g) % p
        return self._make_key(mk(), mk())

    def switch(self, key, digits_dev, path=None):
        """digits_dev: (B, L, N) int64 residues; returns (B, 2, L, N)
        coefficients.  path: "aux" (default when available) or "direct"."""
        torch = self._torch
        B = digits_dev.shape[0]
        out = torch.empty((B, 2, self.L, self.n), dtype=torch.int64, device="cuda")
        use_aux = (path or ("aux" if self.aux else "direct")) == "aux"
        if use_aux:
            if key.aux is None:
                raise ValueError("key has no aux-basis form")
            T = len(self.aux_primes)
            scratch = torch.empty((B * 3 * self.L * T * self.n,), dtype=torch.int32, device="cuda")
            nat.call("hefv_keyswitch64_aux", self._h, key.aux.data_ptr(), digits_dev.data_ptr(),
                     out.data_ptr(), scratch.data_ptr(), B, nat.stream_handle())
        else:
            scratch = torch.empty((B, self.L, self.L, self.n), dtype=torch.int64, device="cuda")
            nat.call("hefv_keyswitch64", self._h, key.mont[0].data_ptr(), key.mont[1].data_ptr(),
                     digits_dev.data_ptr(), out.data_ptr(), scratch.data_ptr(), B,
                     nat.stream_handle())
        return out

    def switch_host(self, key, digits, path=None):
        d = self._dev(np.asarray(digits, dtype=object).astype(np.uint64))
        return nat.to_host(self.switch(key, d.view(-1, self.L, self.n), path)).astype(object)
