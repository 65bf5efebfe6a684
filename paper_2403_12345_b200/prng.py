"""Host side of the particle random-number streams.

The generator is the reference's 63-bit LCG (eventmc/prng.py:1-87):
``s' = (A*s + 1) mod 2**63``, ``u = s * 2**-63`` (pinned to 1-2**-53 if the
float rounds up to 1).  Particle (batch b, index g) owns the window starting
``(b*P + g) * STRIDE`` draws into the master stream; batch-level draws
(resampling) come from ``2**62 + b*STRIDE``.  The device engine evaluates
the same layout in u64 arithmetic (csrc/emc_device.cuh lcg_skip/draw).

``uniform_sequence`` is a vectorised (numpy) form of the sequential draw used
by the library generator: s_k = A^k s_0 + (1 + A + ... + A^{k-1}) evaluated
with wrapping uint64 products and sums, then reduced mod 2**63.
"""

from __future__ import annotations

import numpy as np

MODULUS = 1 << 63
MULTIPLIER = 2806196910506780709
INCREMENT = 1
STRIDE = 152917
AUX_STREAM_OFFSET = 1 << 62

_MASK = MODULUS - 1
_SCALE = 2.0 ** -63
_LAST_BELOW_ONE = 1.0 - 2.0 ** -53


def next_uniform(state: int) -> tuple[float, int]:
    """One step of the generator: returns (u, new_state)."""
    nxt = (MULTIPLIER * state + INCREMENT) & _MASK
    u = nxt * _SCALE
    return (_LAST_BELOW_ONE if u >= 1.0 else u), nxt


def skip_ahead(state: int, n: int) -> int:
    """State after n steps in O(log n) via (mult, add) squaring."""
    if n < 0:
        raise ValueError("skip count must be non-negative")
    n &= _MASK
    mul, add = 1, 0
    step_mul, step_add = MULTIPLIER, INCREMENT
    while n:
        if n & 1:
            mul = (mul * step_mul) & _MASK
            add = (add * step_mul + step_add) & _MASK
        step_add = (step_add * (step_mul + 1)) & _MASK
        step_mul = (step_mul * step_mul) & _MASK
        n >>= 1
    return (mul * state + add) & _MASK


def seed_stream(master_seed: int, batch_index: int, particle_index: int,
                particles_per_batch: int) -> int:
    """First state of the stream of particle (batch, index)."""
    window = batch_index * particles_per_batch + particle_index
    return skip_ahead(master_seed & _MASK, window * STRIDE)


def batch_stream(master_seed: int, batch_index: int) -> int:
    """Stream for batch-level draws (fission-bank resampling)."""
    return skip_ahead(master_seed & _MASK,
                      AUX_STREAM_OFFSET + batch_index * STRIDE)


def uniform_sequence(state: int, n: int) -> np.ndarray:
    """The next n uniforms after `state`, vectorised and bit-identical to n
    sequential next_uniform calls (u64 -> f64 conversion rounds to nearest,
    as the compiled reference does)."""
    if n <= 0:
        return np.empty(0, np.float64)
    with np.errstate(over="ignore"):
        powers = np.cumprod(np.full(n, MULTIPLIER, dtype=np.uint64),
                            dtype=np.uint64)                      # A^1..A^n
        geo = np.empty(n, np.uint64)                               # 1+A+..+A^{k-1}
        geo[0] = 1
        if n > 1:
            geo[1:] = np.cumsum(powers[:-1], dtype=np.uint64) + np.uint64(1)
        states = powers * np.uint64(state & _MASK) + geo
    states &= np.uint64(_MASK)
    u = states.astype(np.float64) * _SCALE
    u[u >= 1.0] = _LAST_BELOW_ONE
    return u
