"""Coarse-grained systems: the SystemSpec container and the synthetic
generators (coil / helix / globule) of the reference (systems.py:40-199).

The generators are host-side input preparation.  They must reproduce the
reference's coordinates bit for bit because the benchmark stand-in for 1ENH
is generate_system("coil", 269, 0); the numpy operation
sequence therefore follows the reference exactly and is pinned by
tests/test_host.py (hash-pinned: test_init_params_bit_identical, test_generate_system_bit_identical, test_quantize_model_bit_identical).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .prior import PriorSpec

DEFAULT_BOND_K = 1000.0   # kJ/(mol nm^2)
DEFAULT_BOND_R0 = 0.38    # nm
DEFAULT_MASS = 110.0      # amu
GENERATOR_TYPES = 8


class SystemFileError(ValueError):
    pass


@dataclass
class SystemSpec:
    types: np.ndarray
    masses: np.ndarray
    prior: PriorSpec | None
    positions: np.ndarray | None
    native: np.ndarray | None
    energy_unit: str = "kJ/mol"

    @property
    def n_beads(self) -> int:
        return int(self.types.size)

    def initial_positions(self) -> np.ndarray:
        for cand in (self.positions, self.native):
            if cand is not None:
                return cand
        raise SystemFileError("system has neither initial nor native coordinates")


def chain_prior(n: int, k: float = DEFAULT_BOND_K, r0: float = DEFAULT_BOND_R0) -> PriorSpec:
    i = np.arange(n - 1)
    return PriorSpec(bonds=np.stack([i, i + 1], axis=1), spring_k=np.full(n - 1, k),
                     rest_length=np.full(n - 1, r0))


def gen_coil(n: int, seed: int) -> np.ndarray:
    """Self-avoiding-ish random walk with fixed bond length (systems.py:144-156)."""
    rng = np.random.default_rng(seed)
    pos = np.zeros((n, 3))
    for i in range(1, n):
        for _attempt in range(64):
            v = rng.normal(size=3)
            v *= DEFAULT_BOND_R0 / np.linalg.norm(v)
            cand = pos[i - 1] + v
            if i < 2:
                break
            if np.min(np.linalg.norm(pos[:i - 1] - cand, axis=1)) > 0.3:
                break
        pos[i] = cand
    return pos


def gen_helix(n: int, seed: int = 0) -> np.ndarray:
    """CG alpha-helix-like spiral (systems.py:159-165)."""
    radius, rise, turn = 0.23, 0.15, math.radians(100.0)
    k = np.arange(n)
    return np.stack([radius * np.cos(turn * k), radius * np.sin(turn * k), rise * k], axis=1)


def gen_globule(n: int, seed: int) -> np.ndarray:
    """Random ball relaxed to a 0.3 nm minimum separation (systems.py:168-185)."""
    rng = np.random.default_rng(seed)
    radius = 0.28 * max(n, 2) ** (1.0 / 3.0)
    pos = rng.normal(size=(n, 3))
    scale = radius * rng.uniform(0, 1, n) ** (1.0 / 3.0) / np.linalg.norm(pos, axis=1)
    pos *= scale[:, None]
    for _ in range(60):
        diff = pos[:, None, :] - pos[None, :, :]
        dist = np.sqrt(np.einsum("ijk,ijk->ij", diff, diff))
        np.fill_diagonal(dist, 1e9)
        close = dist < 0.3
        if not close.any():
            break
        push = np.where(close, (0.3 - dist) / np.maximum(dist, 1e-9), 0.0)
        pos += 0.5 * np.einsum("ij,ijk->ik", push, diff)
    return pos


_MAKERS = {"coil": gen_coil, "helix": gen_helix, "globule": gen_globule}


def generate_system(kind: str, n: int, seed: int, bonded: bool = True) -> SystemSpec:
    if kind not in _MAKERS:
        raise SystemFileError(f"unknown system kind {kind!r}; pick one of {sorted(_MAKERS)}")
    pos = _MAKERS[kind](n, seed)
    types = np.random.default_rng(seed + 1).integers(0, GENERATOR_TYPES, size=n)
    return SystemSpec(types=types, masses=np.full(n, DEFAULT_MASS),
                      prior=chain_prior(n) if bonded and n > 1 else None,
                      positions=pos, native=pos.copy())


def skewed_segments(n_segments: int, n_edges: int, kind: str):
    """Segment-size layouts for degree-skew experiments at a fixed edge count
    (systems.py:202-221): "uniform" spreads edges evenly, "powerlaw" gives
    Zipf(1.1) sizes with the remainder on the head.  Returns (ptr, dst)."""
    if kind == "uniform":
        sizes = np.full(n_segments, n_edges // n_segments, dtype=np.int64)
        sizes[:n_edges % n_segments] += 1
    elif kind == "powerlaw":
        w = 1.0 / np.arange(1, n_segments + 1, dtype=np.float64) ** 1.1
        sizes = np.floor(w / w.sum() * n_edges).astype(np.int64)
        sizes[0] += n_edges - sizes.sum()
    else:
        raise ValueError(f"unknown layout kind {kind!r}")
    ptr = np.zeros(n_segments + 1, dtype=np.int64)
    np.cumsum(sizes, out=ptr[1:])
    return ptr, np.repeat(np.arange(n_segments, dtype=np.int64), sizes)
