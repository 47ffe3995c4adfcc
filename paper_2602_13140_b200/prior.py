"""Harmonic bond prior (reference md.py:90-124) and its device form."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class PriorSpec:
    """Harmonic bonds: E = sum 1/2 k (|r_i - r_j| - r0)^2."""

    bonds: np.ndarray
    spring_k: np.ndarray
    rest_length: np.ndarray

    def __post_init__(self):
        b = np.asarray(self.bonds)
        if b.size and (np.any(b[:, 0] == b[:, 1]) or np.any(np.asarray(self.spring_k) < 0)
                       or np.any(np.asarray(self.rest_length) <= 0)):
            raise ValueError("bonds need i != j, k >= 0 and r0 > 0")

    @property
    def num_bonds(self) -> int:
        return int(np.asarray(self.bonds).shape[0])


def incidence(prior: PriorSpec | None, n: int):
    """Per-bead bond lists in the order np.add.at applies them (md.py:122-123):
    first every bond whose first atom is the bead (sign +1), then every bond
    whose second atom is the bead (sign -1), each in bond order."""
    if prior is None or prior.num_bonds == 0:
        return (np.zeros(n + 1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32))
    b = np.asarray(prior.bonds, dtype=np.int64)
    m = b.shape[0]
    atoms = np.concatenate([b[:, 0], b[:, 1]])
    bond = np.concatenate([np.arange(m), np.arange(m)])
    sign = np.concatenate([np.ones(m, np.int32), -np.ones(m, np.int32)])
    # stable sort by atom keeps the (+ pass, - pass) x bond order within a bead
    order = np.argsort(atoms, kind="stable")
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(atoms, minlength=n), out=ptr[1:])
    return ptr.astype(np.int32), bond[order].astype(np.int32), sign[order]


class DevicePrior:
    def __init__(self, prior: PriorSpec | None, n: int, device="cuda"):
        import torch

        self._keep = []

        def dev(a, dt):
            t = torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=dt)
            self._keep.append(t)
            return t

        ptr, bond, sign = incidence(prior, n)
        d = _lib.FcgPrior()
        d.num_bonds = 0 if prior is None else prior.num_bonds
        if d.num_bonds:
            b = np.asarray(prior.bonds, dtype=np.int32)
            d.bond_i = _lib.i32ptr(dev(b[:, 0], torch.int32))
            d.bond_j = _lib.i32ptr(dev(b[:, 1], torch.int32))
            d.k = _lib.fptr(dev(np.asarray(prior.spring_k).astype(np.float32), torch.float32))
            d.r0 = _lib.fptr(dev(np.asarray(prior.rest_length).astype(np.float32), torch.float32))
            d.inc_bond = _lib.i32ptr(dev(bond, torch.int32))
            d.inc_sign = _lib.i32ptr(dev(sign, torch.int32))
        d.inc_ptr = _lib.i32ptr(dev(ptr, torch.int32))
        self.desc = d
