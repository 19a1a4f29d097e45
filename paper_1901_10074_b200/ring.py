"""Host-side number theory: prime search, primitive roots, CRT constants.

Only the once-per-context integer precompute lives here -- every transform
and every per-coefficient computation runs in libhefv.so.  The choices must
reproduce the reference exactly, because they fix the residues:

* ``find_ntt_primes`` walks candidates p = 1 (mod 2N) downward from 2^bits
  (reference ntt.py:115-131), including the ``below`` rule used for the
  auxiliary basis (fv.py:89-95);
* psi = g^((p-1)/2N) with g the *smallest* generator (ntt.py:105-112,
  ntt.py:155-156) -- any other root permutes evaluation points;
* q primes: max(2, ceil(coeff_modulus_bits / 30)) primes of 30 bits
  (fv.py:60-64); aux primes: ceil((bitlen N + 2 bitlen q + 2) / 29) primes
  below min(q) (fv.py:89-95).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

WORD_BITS = 30
_MR_WITNESSES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (exact for n < 3.3e24)."""
    if n < 2:
        return False
    for w in _MR_WITNESSES:
        if n % w == 0:
            return n == w
    d, r = n - 1, 0
    while not d & 1:
        d >>= 1
        r += 1
    for w in _MR_WITNESSES:
        x = pow(w, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _prime_factors(n: int) -> list:
    out, f = [], 2
    while f * f <= n:
        if n % f == 0:
            out.append(f)
            while n % f == 0:
                n //= f
        f += 1 if f == 2 else 2
    if n > 1:
        out.append(n)
    return out


@lru_cache(maxsize=None)
def primitive_root(p: int) -> int:
    """Smallest generator of (Z/p)^*."""
    factors = _prime_factors(p - 1)
    g = 2
    while any(pow(g, (p - 1) // f, p) == 1 for f in factors):
        g += 1
    return g


def find_ntt_primes(count: int, bits: int, two_n: int, below=None) -> list:
    """``count`` primes p = 1 (mod two_n), walking down from 2^bits."""
    cand = (1 << bits) // two_n * two_n + 1
    if below is not None:
        cand = min(cand, (below - 2) // two_n * two_n + 1)
    found = []
    while len(found) < count:
        if cand < two_n:
            raise ValueError("ran out of candidate primes")
        if is_prime(cand):
            found.append(cand)
        cand -= two_n
    return found


def root_of_unity(p: int, n: int) -> int:
    """psi: the primitive 2n-th root the reference's NttPrime uses."""
    if (p - 1) % (2 * n):
        raise ValueError(f"p={p} is not 1 mod {2 * n}")
    return pow(primitive_root(p), (p - 1) // (2 * n), p)


def bitrev_perm(log_n: int) -> np.ndarray:
    """i -> bitrev(i) over log_n bits."""
    n = 1 << log_n
    idx = np.arange(n, dtype=np.int64)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(log_n):
        rev |= ((idx >> b) & 1) << (log_n - 1 - b)
    return rev


def to_words(x: int, w: int) -> np.ndarray:
    """Little-endian 32-bit words of a non-negative integer."""
    if x < 0 or x >> (32 * w):
        raise ValueError("value does not fit the word count")
    return np.array([(x >> (32 * i)) & 0xFFFFFFFF for i in range(w)], dtype=np.uint32)


def words_for(x: int) -> int:
    return max(1, -(-x.bit_length() // 32))


@dataclass
class CrtConstants:
    """CRT interpolation constants for a basis P = prod p_i."""

    primes: list
    product: int
    words: int
    prod_words: np.ndarray
    half_words: np.ndarray
    hat_words: np.ndarray  # (len, words): P / p_i
    hat_inv: np.ndarray    # (len,): (P / p_i)^-1 mod p_i

    @classmethod
    def build(cls, primes, words=None) -> "CrtConstants":
        prod = 1
        for p in primes:
            prod *= p
        w = words or words_for(prod)
        hats = [prod // p for p in primes]
        return cls(
            primes=list(primes),
            product=prod,
            words=w,
            prod_words=to_words(prod, w),
            half_words=to_words(prod // 2, w),
            hat_words=np.stack([to_words(h, w) for h in hats]) if primes else np.zeros((0, w), np.uint32),
            hat_inv=np.array([pow(h % p, -1, p) for h, p in zip(hats, primes)], dtype=np.uint32),
        )


def slot_to_eval(n: int) -> np.ndarray:
    """Slot i <-> natural evaluation index (3^i mod 2n - 1) / 2 (fv.py:102-109)."""
    exps = np.empty(n // 2, dtype=np.int64)
    e = 1
    for i in range(n // 2):
        exps[i] = e
        e = e * 3 % (2 * n)
    return (exps - 1) // 2


def galois_element(offset: int, n: int) -> int:
    """x -> x^(3^offset mod 2n) rotates slots left by ``offset`` (fv.py:427)."""
    return pow(3, offset, 2 * n)


def gadget(q_primes) -> list:
    """g_i = (q/q_i) * ((q/q_i)^-1 mod q_i) mod q (fv.py:97-100), as ints."""
    q = 1
    for p in q_primes:
        q *= p
    return [(q // p) * pow(q // p, -1, p) % q for p in q_primes]
