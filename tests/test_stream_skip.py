"""The device's per-particle stream start (csrc/emc_device.cuh lcg_gskip):
the batch base lcg_skip(seed, b*P*STRIDE), computed on the host once per
batch, advanced by g*STRIDE through a table of the affine maps of
STRIDE*2^j -- must equal the reference's seed_stream (prng.py:54-58) for
every (seed, batch, g), including offsets past 2^63.  CPU restatement of the
device arithmetic; the GPU parity suite checks the kernels themselves."""
import random

from paper_2403_12345_b200 import prng

MASK = prng.MODULUS - 1


def table():
    tab = []
    for j in range(64):
        n = ((prng.STRIDE << j) & MASK) if j < 63 else 0
        aa = prng.skip_ahead(0, n)
        tab.append(((prng.skip_ahead(1, n) - aa) & MASK, aa))
    return tab


def gskip(tab, s, g):
    j = 0
    while g:
        if g & 1:
            s = (tab[j][0] * s + tab[j][1]) & MASK
        g >>= 1
        j += 1
    return s


def test_table_skip_equals_seed_stream():
    tab = table()
    rng = random.Random(7)
    cases = [(42, 0, 40_000_000, 0), (42, 24, 40_000_000, 39_999_999), (0, 0, 1, 0), (MASK, 3, 10, 9),
             (12345, 2 ** 20, 2 ** 40, 2 ** 40 - 1)]
    for _ in range(300):
        p = rng.randrange(1, 2 ** rng.randrange(1, 40))
        cases.append((rng.randrange(2 ** 64), rng.randrange(2 ** 16), p, rng.randrange(p)))
    for seed, b, p, g in cases:
        base = prng.skip_ahead(seed & MASK, ((b * p) * prng.STRIDE) % 2 ** 64)
        assert gskip(tab, base, g) == prng.seed_stream(seed, b, g, p), (seed, b, p, g)
