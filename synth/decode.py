"""Seeded inputs for the f1 decode-loop tests and bench: bf16 query / new-token K,V tensors and
ragged sequence lengths. Holds none of the method's arithmetic (input generation only)."""
from __future__ import annotations

import numpy as np


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float -> bf16 bits, round to nearest even (input generation only)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def gaussian_bf16(rng: np.random.Generator, shape, scale: float = 1.0) -> np.ndarray:
    return bf16_bits(rng.standard_normal(shape).astype(np.float32) * np.float32(scale))


def ragged_lengths(rng: np.random.Generator, n: int, max_len: int) -> np.ndarray:
    """Lengths that hit the edge cases (0, 1, d-1, d, d+1, chunk boundaries) then random ones."""
    edge = [0, 1, 15, 16, 17, 255, 256, 257]
    out = [e for e in edge if e <= max_len][:n]
    out += list(rng.integers(1, max_len + 1, max(0, n - len(out))))
    return np.asarray(out, np.int32)
