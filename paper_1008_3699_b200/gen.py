"""Seeded synthetic input generators (shared by tests, bench and the oracle harness).

This module holds NO arithmetic of the method (no stencil, no sweep, no face
averaging).  It only draws the raw fields the paper's model problems are made of:

* ``uniform(seed, stream, count)``  -> U[-1, 1) fp64 (right-hand sides, PAPER:1906-1934
  uses f = 0; BASELINE.json configs use f ~ U[-1,1]).
* ``normal(seed, stream, count)``   -> N(0, 1) fp64 (log-diffusivity for configs 3 and 5).

Generator: counter-based splitmix64 (SURVEY.md §8(c) c-amb-13).  Element ``i`` of
stream ``s`` is ``splitmix64(seed * 0x9E3779B97F4A7C15 + (s << 40) + i)``, so any slab
of any array can be generated independently on any rank.  Uniform values use the top
53 bits; normals use Box-Muller on two consecutive uniform draws.
"""
from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# stream ids (fixed so every consumer draws the same numbers)
STREAM_RHS = 1
STREAM_LOGK = 2
STREAM_X0 = 3
STREAM_TEST = 7


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _counters(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * _GOLD + (np.uint64(stream) << np.uint64(40)) + np.uint64(start)
        return base + np.arange(count, dtype=np.uint64)


def unit(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """U[0,1) with 53-bit resolution."""
    bits = _splitmix64(_counters(seed, stream, start, count))
    return (bits >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """U[-1,1)."""
    return 2.0 * unit(seed, stream, count, start) - 1.0


def normal(seed: int, stream: int, count: int, start: int = 0) -> np.ndarray:
    """N(0,1) via Box-Muller on draws (2i, 2i+1)."""
    u = unit(seed, stream, 2 * count, 2 * start)
    u1 = 1.0 - u[0::2]          # (0, 1]
    u2 = u[1::2]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def uniform_field(seed: int, stream: int, shape, start: int = 0) -> np.ndarray:
    count = int(np.prod(shape))
    return uniform(seed, stream, count, start).reshape(shape)


def normal_field(seed: int, stream: int, shape, start: int = 0) -> np.ndarray:
    count = int(np.prod(shape))
    return normal(seed, stream, count, start).reshape(shape)


def lognormal_k(seed: int, shape_with_ring, sigma: float) -> np.ndarray:
    """Node diffusivity k = exp(sigma * N(0,1)) on all nodes INCLUDING the boundary ring.

    Config 3: sigma = 1 on 4098^2 nodes; config 5: sigma = 0.5 on 514^3 nodes
    (SURVEY.md §8(c) c-amb-12).  Shape is given slow-axis first (z, y, x).
    """
    return np.exp(sigma * normal_field(seed, STREAM_LOGK, shape_with_ring))
