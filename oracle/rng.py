"""CPU restatement of the numpy random primitives the reference search depends on.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the checker. The product path never calls it.

The reference (pure Python) draws its search seeds through numpy 2.3.5
(third-party, pinned here; not vendored under /root/reference):

* ``derive_query_seed`` -- ``SeedSequence([seed, ordinal]).generate_state(1, u64)``
  (reference pkg/src/bucketann/searcher.py:85-87);
* ``default_rng(seed)`` -> PCG64 seeded through ``SeedSequence(seed)``
  (searcher.py:181);
* ``rng.integers(0, total, size)`` -> Lemire bounded 32-bit draws over the
  buffered 32-bit PCG64 output (searcher.py:128).

This module restates the published algorithms (O'Neill PCG-XSL-RR-128/64,
numpy's SeedSequence hash mixer, Lemire 2018 nearly-divisionless bounded ints)
with plain Python integers, so the CUDA restatement in
paper_2604_16402_b200/csrc/rng.cuh has a readable twin. tests/test_oracle_rng.py
pins it against numpy itself.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
M128 = (1 << 128) - 1

# SeedSequence hash constants (numpy/random/bit_generator.pyx)
_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_POOL = 4

# PCG64 default 128-bit LCG multiplier
PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341


def int_words(v: int) -> list[int]:
    """Little-endian 32-bit words of a non-negative int; 0 -> [0]."""
    if v < 0:
        raise ValueError("seed entropy must be non-negative")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & M32)
        v >>= 32
    return out


def seedseq_pool(entropy: list[int]) -> list[int]:
    """Mix the entropy words into the 4-word pool."""
    words: list[int] = []
    for e in entropy:
        words.extend(int_words(e))
    hc = _INIT_A

    def hashmix(v: int) -> int:
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * _MULT_A) & M32
        v = (v * hc) & M32
        return v ^ (v >> 16)

    def mix(x: int, y: int) -> int:
        r = (_MIX_L * x - _MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(_POOL)]
    for s in range(_POOL):
        for d in range(_POOL):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(_POOL, len(words)):
        for d in range(_POOL):
            pool[d] = mix(pool[d], hashmix(words[s]))
    return pool


def seedseq_words(pool: list[int], n_words32: int) -> list[int]:
    hc = _INIT_B
    out = []
    for i in range(n_words32):
        v = (pool[i % _POOL] ^ hc) & M32
        hc = (hc * _MULT_B) & M32
        v = (v * hc) & M32
        out.append(v ^ (v >> 16))
    return out


def seedseq_u64(entropy: list[int], n: int) -> list[int]:
    w = seedseq_words(seedseq_pool(entropy), 2 * n)
    return [w[2 * i] | (w[2 * i + 1] << 32) for i in range(n)]


def derive_query_seed(base: int, ordinal: int) -> int:
    """searcher.py:85-87 restated."""
    return seedseq_u64([base, ordinal], 1)[0]


class PCG64:
    """XSL-RR 128/64 with numpy's buffered 32-bit output (low half first)."""

    def __init__(self, seed: int):
        v = seedseq_u64([seed], 4)
        initstate = (v[0] << 64) | v[1]
        initseq = (v[2] << 64) | v[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()
        self._buf = None

    def _step(self) -> None:
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self) -> int:
        self._step()
        s = self.state
        x = ((s >> 64) ^ s) & M64
        r = s >> 122
        return ((x >> r) | (x << ((64 - r) & 63))) & M64

    def next32(self) -> int:
        if self._buf is not None:
            v, self._buf = self._buf, None
            return v
        x = self.next64()
        self._buf = x >> 32
        return x & M32

    def integers(self, total: int, size: int) -> list[int]:
        """``Generator.integers(0, total, size)`` for 1 <= total <= 2**32 - 1."""
        if total == 1:
            return [0] * size
        thresh = ((1 << 32) - total) % total
        out = []
        for _ in range(size):
            while True:
                m = self.next32() * total
                if (m & M32) >= thresh:
                    break
            out.append(m >> 32)
        return out
