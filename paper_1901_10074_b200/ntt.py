"""GPU-backed drop-in for the reference's ``hepack.ntt`` module.

``NttPrime(p, n).fwd/inv/negacyclic_mul`` keep the reference's semantics
(/root/reference/pkg/src/hepack/ntt.py:142-227): natural-order evaluations
fwd(a)[k] = a(psi^(2k+1)) with the reference's choice of psi, batched over
leading axes -- but every transform runs in libhefv.so (30-bit primes on
the 32-bit kernels, primes up to 2^62 on the 64-bit kernels).  Prime search
and CRT interpolation constants are host integer precompute (ring.py).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from .ring import find_ntt_primes, is_prime, primitive_root, root_of_unity  # noqa: F401

__all__ = ["NttPrime", "CrtBasis", "find_ntt_primes", "is_prime", "primitive_root"]

_U32_LIMIT = 1 << 30
_U64_LIMIT = 1 << 62


class NttPrime:
    """Negacyclic NTT tables for one prime p = 1 (mod 2n), on the device."""

    def __init__(self, p: int, n: int):
        import ctypes as C

        import torch

        if (p - 1) % (2 * n) != 0:
            raise ValueError(f"p={p} is not 1 mod {2 * n}")
        if n < 2 or n > 1 << 16 or n & (n - 1):
            raise ValueError("ring dimension must be a power of two in [2, 65536]")
        if p >= _U64_LIMIT:
            raise ValueError("primes must be below 2^62")
        nat.require_device()
        lib = nat.load()
        self.p = p
        self.n = n
        self.log_n = n.bit_length() - 1
        self.psi = root_of_unity(p, n)
        self.dtype = np.int64 if p < (1 << 31) else object
        self.wide = p >= _U32_LIMIT or (self.log_n == 16)
        h = C.c_void_p()
        if self.wide:
            pr = (C.c_uint64 * 1)(p)
            ps = (C.c_uint64 * 1)(self.psi)
            nat.check(lib.hefv_ctx_create(C.byref(h), self.log_n, 0, None, None, 1, pr, ps),
                      "hefv_ctx_create")
        else:
            pr = (C.c_uint32 * 1)(p)
            ps = (C.c_uint32 * 1)(self.psi)
            nat.check(lib.hefv_ctx_create(C.byref(h), self.log_n, 1, pr, ps, 0, None, None),
                      "hefv_ctx_create")
        self._h = h
        self._torch = torch

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and nat._lib is not None:
            nat._lib.hefv_ctx_destroy(h)
            self._h = None

    def _upload(self, a):
        torch = self._torch
        arr = np.asarray(a)
        if arr.shape[-1] != self.n:
            raise ValueError(f"last axis must be {self.n}")
        lead = arr.shape[:-1]
        flat = arr.reshape(-1, self.n)
        # host-side normalisation of arbitrary integers into [0, p) (input coercion only)
        if flat.dtype == object or (flat.dtype.kind in "iu" and flat.dtype.itemsize > 8):
            flat = np.array([[int(v) % self.p for v in row] for row in flat], dtype=np.uint64)
        else:
            flat = np.mod(flat.astype(np.int64), self.p).astype(np.uint64)
        if self.wide:
            dev = torch.from_numpy(flat.view(np.int64)).cuda()
        else:
            dev = torch.from_numpy(flat.astype(np.int32)).cuda()
        return dev, lead

    def _transform(self, dev, forward: bool):
        out = self._torch.empty_like(dev)
        if self.wide:
            fn = "hefv_ntt_fwd64" if forward else "hefv_ntt_inv64"
        else:
            fn = "hefv_ntt_fwd32" if forward else "hefv_ntt_inv32"
        nat.call(fn, self._h, dev.data_ptr(), out.data_ptr(), dev.shape[0], 1, 0, 1,
                 nat.stream_handle())
        return out

    def _download(self, dev, lead) -> np.ndarray:
        res = dev.cpu().numpy().astype(np.int64).reshape(*lead, self.n)
        return res.astype(object) if self.dtype is object else res

    def _run(self, a, forward: bool) -> np.ndarray:
        dev, lead = self._upload(a)
        return self._download(self._transform(dev, forward), lead)

    def fwd(self, a) -> np.ndarray:
        """Evaluations at the odd powers of psi, natural order (ntt.py:216-219)."""
        return self._run(a, True)

    def inv(self, ev) -> np.ndarray:
        """Inverse of fwd (ntt.py:221-224)."""
        return self._run(ev, False)

    def negacyclic_mul(self, a, b) -> np.ndarray:
        """Ring product mod (x^N + 1, p) (ntt.py:226-227): both transforms,
        the pointwise product and the inverse on the device."""
        da, lead = self._upload(a)
        db, lead_b = self._upload(b)
        if lead != lead_b:
            raise ValueError("operands must have the same shape")
        fa = self._transform(da, True)
        fb = self._transform(db, True)
        prod = self._torch.empty_like(fa)
        nat.call("hefv_pointwise_mul", self._h, 1 if self.wide else 0, fa.data_ptr(),
                 fb.data_ptr(), prod.data_ptr(), fa.shape[0], 1, 0, nat.stream_handle())
        return self._download(self._transform(prod, False), lead)


class CrtBasis:
    """Residues <-> integers for a prime basis (ntt.py:248-271).

    Host utility kept for API compatibility (the device path reconstructs
    inside the multiprecision kernels)."""

    def __init__(self, primes):
        self.primes = list(primes)
        self.product = 1
        for p in self.primes:
            self.product *= p
        self._interp = np.array(
            [(self.product // p) * pow(self.product // p, -1, p) % self.product for p in self.primes],
            dtype=object)

    def to_big(self, residues: np.ndarray) -> np.ndarray:
        return residues.astype(object).T @ self._interp % self.product

    def from_big(self, values) -> np.ndarray:
        values = np.asarray(values, dtype=object)
        return np.stack([(values % p).astype(np.int64) for p in self.primes])
