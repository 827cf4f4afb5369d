"""Random streams for the oracle (test infrastructure only, see oracle/__init__).

Reference behaviour restated here:
  * `mix64` — splitmix64-style fold of integer parts  (engine.py:74-83)
  * `derived_rng(*parts)` = `random.Random(mix64(*parts))` (engine.py:86-87);
    stream discriminators lane/accept/init/migration/probe (engine.py:67-71).
  * The draws operators make go through CPython's `random.Random` methods:
    `random()` (two 32-bit words, 53-bit mantissa), `randrange()` ->
    `_randbelow_with_getrandbits` (k = n.bit_length(), rejection), `shuffle`
    (Fisher-Yates from the top), `sample` (pool or set method).

`WordRandom` re-implements exactly those methods on top of an arbitrary
32-bit word source, so that

    WordRandom(mt_words(seed))      == random.Random(seed)      (checked in tests)
    WordRandom(philox_words(key))   == the GPU lane stream      (checked on GPU)

i.e. the GPU engine consumes the reference's draw sequence with Philox4x32-10
words in place of MT19937 words.
"""

from __future__ import annotations

import math
import random

MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1

STREAM_LANE = 0
STREAM_ACCEPT = 1
STREAM_INIT = 2
STREAM_MIGRATION = 3
STREAM_PROBE = 4


def mix64(*parts: int) -> int:
    """engine.py:74-83 — fold each part into a splitmix64 finaliser."""
    h = 0x9E3779B97F4A7C15
    for part in parts:
        h = (h ^ (part & MASK64)) & MASK64
        h = (h * 0xBF58476D1CE4E5B9) & MASK64
        h ^= h >> 27
        h = (h * 0x94D049BB133111EB) & MASK64
        h ^= h >> 31
    return h


# ---------------------------------------------------------------------------
# Philox4x32-10 (Salmon et al., SC'11; Random123 constants)

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85


def philox4x32_10(ctr, key):
    """One Philox4x32-10 block: 4 x uint32 counter, 2 x uint32 key -> 4 words."""
    c0, c1, c2, c3 = (int(c) & MASK32 for c in ctr)
    k0, k1 = int(key[0]) & MASK32, int(key[1]) & MASK32
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W0) & MASK32
            k1 = (k1 + PHILOX_W1) & MASK32
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0, p1 & MASK32,
                          (p0 >> 32) ^ c3 ^ k1, p0 & MASK32)
    return c0, c1, c2, c3


class PhiloxWords:
    """Word source of one GPU lane stream: key = 64-bit stream hash,
    counter = (block index, 0, 0, 0); words are consumed 0..3 per block."""

    __slots__ = ("k0", "k1", "block", "buf", "at")

    def __init__(self, key64: int):
        self.k0 = key64 & MASK32
        self.k1 = (key64 >> 32) & MASK32
        self.block = 0
        self.buf = ()
        self.at = 4

    def __call__(self) -> int:
        if self.at == 4:
            self.buf = philox4x32_10((self.block, 0, 0, 0), (self.k0, self.k1))
            self.block += 1
            self.at = 0
        w = self.buf[self.at]
        self.at += 1
        return w


def mt_words(seed: int):
    """MT19937 word source identical to random.Random(seed).getrandbits(32)."""
    gen = random.Random(seed)
    return lambda: gen.getrandbits(32)


class WordRandom:
    """CPython `random.Random` draw algorithms over a 32-bit word source."""

    __slots__ = ("word", "words_used")

    def __init__(self, word):
        self.word = word
        self.words_used = 0

    def _w(self) -> int:
        self.words_used += 1
        return self.word()

    def getrandbits(self, k: int) -> int:
        if k <= 0:
            return 0
        if k > 32:
            raise ValueError("oracle streams only draw <= 32 bits at a time")
        return self._w() >> (32 - k)

    def random(self) -> float:
        a = self._w() >> 5
        b = self._w() >> 6
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0)

    def _randbelow(self, n: int) -> int:
        k = n.bit_length()
        r = self.getrandbits(k)
        while r >= n:
            r = self.getrandbits(k)
        return r

    def randrange(self, start: int, stop: int | None = None) -> int:
        if stop is None:
            if start > 0:
                return self._randbelow(start)
            raise ValueError("empty range for randrange()")
        width = stop - start
        if width > 0:
            return start + self._randbelow(width)
        raise ValueError(f"empty range in randrange({start}, {stop})")

    def shuffle(self, x) -> None:
        for i in range(len(x) - 1, 0, -1):
            j = self._randbelow(i + 1)
            x[i], x[j] = x[j], x[i]

    def sample(self, population, k: int):
        n = len(population)
        if not 0 <= k <= n:
            raise ValueError("Sample larger than population or is negative")
        out = [None] * k
        setsize = 21
        if k > 5:
            setsize += 4 ** math.ceil(math.log(k * 3, 4))
        if n <= setsize:
            pool = list(population)
            for i in range(k):
                j = self._randbelow(n - i)
                out[i] = pool[j]
                pool[j] = pool[n - i - 1]
        else:
            chosen = set()
            for i in range(k):
                j = self._randbelow(n)
                while j in chosen:
                    j = self._randbelow(n)
                chosen.add(j)
                out[i] = population[j]
        return out


def mt_stream(*parts: int):
    """The reference's derived_rng (engine.py:86-87)."""
    return random.Random(mix64(*parts))


def philox_stream(*parts: int) -> WordRandom:
    """The GPU engine's stream for the same parts."""
    return WordRandom(PhiloxWords(mix64(*parts)))


STREAMS = {"mt": mt_stream, "philox": philox_stream}
