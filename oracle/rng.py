"""Pure-Python restatement of the numpy RNG pieces the reference path uses
(TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The reference draws randomness only through numpy (numpy 2.3.5 here; the
reference pins ``numpy>=1.24`` at pkg/pyproject.toml:10):
  * ``np.random.default_rng([seed, node]).choice(deg, k, replace=False)``
    (embedding.py:56-57)  -> SeedSequence -> PCG64 -> Floyd's algorithm with
    Lemire bounded 32-bit draws from PCG64's buffered next_uint32;
  * ``np.random.default_rng(seed).random((N, 1))`` (policy.py:235, 288) ->
    PCG64 next_uint64 >> 11 times 2**-53.
The published algorithms (numpy/random/bit_generator.pyx SeedSequence,
numpy/random/src/pcg64, numpy/random/_generator.pyx choice, distributions.c
random_bounded_uint64) are restated here with Python ints so the CUDA
implementation has an independent, readable spec; tests/test_oracle_golden.py
checks them against numpy itself and against the reference's own picks.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1

# SeedSequence constants (bit_generator.pyx)
INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL_SIZE = 4

PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341


def _int_words(x: int) -> list[int]:
    if x < 0:
        raise ValueError("negative entropy")
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & M32)
        x >>= 32
    return out


def seed_words(entropy) -> list[int]:
    if isinstance(entropy, int):
        return _int_words(entropy)
    words = []
    for e in entropy:
        words += _int_words(int(e))
    return words


def seedseq_pool(entropy) -> list[int]:
    ent = seed_words(entropy)
    hc = INIT_A

    def hashmix(value):
        nonlocal hc
        value = (value ^ hc) & M32
        hc = (hc * MULT_A) & M32
        value = (value * hc) & M32
        value ^= value >> XSHIFT
        return value

    def mix(x, y):
        r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
        r ^= r >> XSHIFT
        return r

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(POOL_SIZE)]
    for i_src in range(POOL_SIZE):
        for i_dst in range(POOL_SIZE):
            if i_src != i_dst:
                pool[i_dst] = mix(pool[i_dst], hashmix(pool[i_src]))
    for i_src in range(POOL_SIZE, len(ent)):
        for i_dst in range(POOL_SIZE):
            pool[i_dst] = mix(pool[i_dst], hashmix(ent[i_src]))
    return pool


def seedseq_generate_u64(entropy, n_words64: int) -> list[int]:
    pool = seedseq_pool(entropy)
    hc = INIT_B
    w32 = []
    for i in range(2 * n_words64):
        v = pool[i % POOL_SIZE]
        v = (v ^ hc) & M32
        hc = (hc * MULT_B) & M32
        v = (v * hc) & M32
        v ^= v >> XSHIFT
        w32.append(v)
    return [w32[2 * i] | (w32[2 * i + 1] << 32) for i in range(n_words64)]


class PCG64:
    """numpy's PCG64 (XSL-RR 128/64): step then output the new state."""

    def __init__(self, entropy):
        s = seedseq_generate_u64(entropy, 4)
        initstate = (s[0] << 64) | s[1]
        initseq = (s[2] << 64) | s[3]
        self.inc = ((initseq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + initstate) & M128
        self._step()
        self.has32 = False
        self.buf32 = 0

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    @staticmethod
    def output(state: int) -> int:
        hi, lo = state >> 64, state & M64
        rot = hi >> 58
        x = hi ^ lo
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next64(self) -> int:
        self._step()
        return self.output(self.state)

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.buf32
        v = self.next64()
        self.has32 = True
        self.buf32 = v >> 32
        return v & M32

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def advance(self, delta: int):
        """Jump ahead delta steps (LCG power by squaring)."""
        acc_mult, acc_plus = 1, 0
        cur_mult, cur_plus = PCG_MULT, self.inc
        while delta > 0:
            if delta & 1:
                acc_mult = (acc_mult * cur_mult) & M128
                acc_plus = (acc_plus * cur_mult + cur_plus) & M128
            cur_plus = ((cur_mult + 1) * cur_plus) & M128
            cur_mult = (cur_mult * cur_mult) & M128
            delta >>= 1
        self.state = (acc_mult * self.state + acc_plus) & M128

    def bounded_lemire32(self, rng: int) -> int:
        """distributions.c buffered_bounded_lemire_uint32, inclusive [0, rng]."""
        rng_excl = rng + 1
        m = self.next32() * rng_excl
        left = m & M32
        if left < rng_excl:
            threshold = ((M32 - rng) % rng_excl)
            while left < threshold:
                m = self.next32() * rng_excl
                left = m & M32
        return m >> 32

    def bounded(self, rng: int) -> int:
        """random_bounded_uint64(off=0, rng, use_masked=False) for rng < 2**32."""
        if rng == 0:
            return 0
        if rng == M32:
            return self.next32()
        if rng > M32:
            raise NotImplementedError("64-bit bounded draws are not on the path")
        return self.bounded_lemire32(rng)


def floyd_choice_set(seed: int, node: int, n: int, k: int) -> list[int]:
    """Set chosen by default_rng([seed, node]).choice(n, k, replace=False)
    via Floyd's algorithm (_generator.pyx choice, the non-tail-shuffle branch
    taken whenever not (n > 10000 and k > n // 50)), returned sorted."""
    if n > 10000 and k > n // 50:
        raise NotImplementedError("tail-shuffle branch of Generator.choice")
    g = PCG64([seed, node])
    chosen = set()
    for j in range(n - k, n):
        val = g.bounded(j)
        if val in chosen:
            chosen.add(j)
        else:
            chosen.add(val)
    return sorted(chosen)


def uniform_at(seed: int, index: int) -> float:
    """The index-th double of default_rng(seed).random(...)."""
    g = PCG64(seed)
    g.advance(index)
    return g.random()
