"""Neighbour lists and grouped CSR layouts on the GPU (reference
neighbors.py).  Same types and canonical (dst, src) order; the edge set and
layouts are bit-identical to build_neighbors_cells + group_by_* because the
fp64 cutoff predicate is evaluated with the reference's rounding sequence
(see csrc/nbr.cu)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class NeighborList:
    src: np.ndarray  # int64[E]
    dst: np.ndarray  # int64[E]
    n: int

    @property
    def num_edges(self) -> int:
        return int(self.src.size)


@dataclass(frozen=True)
class CsrLayout:
    ptr: np.ndarray   # int64[N+1]
    perm: np.ndarray  # int64[E]
    key: str          # "dst" | "src"

    @property
    def num_segments(self) -> int:
        return int(self.ptr.size - 1)

    def segment_sizes(self) -> np.ndarray:
        return self.ptr[1:] - self.ptr[:-1]


def _torch():
    from .engine import _torch as t
    return t()


def _stream(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


_CSR_BUFFERS: dict = {}
CAP_LIMIT = 2 ** 31 - 2   # int32 slot indices (include/fcg.h)


def _csr_buffers(torch, n_nodes: int, cap: int):
    """Reusable device CSR buffers per device, grown on demand (never sized
    for the dense R*N*(N-1) worst case)."""
    if cap > CAP_LIMIT:
        raise ValueError(f"neighbour list needs {cap} edge slots; the int32 CSR holds at most "
                         f"{CAP_LIMIT}")
    dev = torch.cuda.current_device()
    b = _CSR_BUFFERS.get(dev)
    if b is None or b["ptr"].numel() < n_nodes + 1 or b["cap"] < cap:
        old_cap = b["cap"] if b is not None else 0
        cap = max(cap, old_cap)
        n_alloc = max(n_nodes + 1, b["ptr"].numel() if b is not None else 0)
        i32 = dict(dtype=torch.int32, device="cuda")
        b = _CSR_BUFFERS[dev] = {
            "cap": cap, "ptr": torch.empty(n_alloc, **i32), "nbr": torch.empty(cap + 1, **i32),
            "rev": torch.empty(cap + 1, **i32), "own": torch.empty(cap + 1, **i32)}
    return b


def device_csr(positions: np.ndarray, r_cut: float, replicas: bool = False):
    """Run fcg_nbr_build on one system ([N,3]) or a replica batch ([R,N,3]).

    Returns (ptr, nbr, rev, own) as int64 numpy arrays over the flattened
    block-diagonal graph.  The edge capacity starts at the engine's
    default (O(R*N), like the reference's O(E) cell list) and grows to the
    built edge count when the build reports an overflow; buffers are reused
    across calls.
    """
    from .engine import default_capacity

    torch = _torch()
    lib = _lib.load()
    pos = np.asarray(positions)
    if pos.ndim == 2:
        pos = pos[None]
    R, N = pos.shape[0], pos.shape[1]
    if N == 0:
        raise ValueError("need at least one bead")
    f64 = pos.dtype == np.float64
    dt = torch.float64 if f64 else torch.float32
    dpos = torch.as_tensor(np.ascontiguousarray(pos, dtype=np.float64 if f64 else np.float32)
                           ).to("cuda", dt)
    status = torch.zeros(_lib.FCG_STATUS_WORDS, dtype=torch.int64, device="cuda")
    nb = lib.fcg_nbr_workspace_bytes(R, N)
    ws = torch.zeros(int(nb), dtype=torch.uint8, device="cuda")  # zero before first use
    fn = lib.fcg_nbr_build_f64 if f64 else lib.fcg_nbr_build
    v = _lib.vp
    cap = default_capacity(R, N)
    while True:
        b = _csr_buffers(torch, R * N, cap)
        ptr, nbr, rev, own = b["ptr"][:R * N + 1], b["nbr"], b["rev"], b["own"]
        _lib.check(fn(v(dpos), R, N, float(r_cut), b["cap"], v(ptr), v(nbr), v(rev), v(own),
                      v(status), v(ws), nb, _stream(torch)), "fcg_nbr_build")
        p = ptr.cpu().numpy().astype(np.int64)
        E = int(p[-1])
        if E <= b["cap"]:
            break
        status.zero_()
        cap = E   # the count pass is exact: one rebuild at this capacity fits
    return (p, nbr[:E].cpu().numpy().astype(np.int64), rev[:E].cpu().numpy().astype(np.int64),
            own[:E].cpu().numpy().astype(np.int64))


def build_neighbors_cells(positions: np.ndarray, r_cut: float) -> NeighborList:
    """Directed cutoff graph, both orientations, canonical (dst, src) order
    (reference neighbors.py:67-110)."""
    pos = np.asarray(positions)
    if pos.shape[0] == 0:
        raise ValueError("need at least one bead")
    _ptr, nbr, _rev, own = device_csr(pos, r_cut)
    return NeighborList(src=nbr, dst=own, n=int(pos.shape[0]))


def build_neighbors_bruteforce(positions: np.ndarray, r_cut: float) -> NeighborList:
    """The reference's O(N^2) oracle (neighbors.py:53-64).  The GPU builder
    is already an exhaustive all-pairs scan, so both names share it."""
    return build_neighbors_cells(positions, r_cut)


def _group(key: np.ndarray, n: int):
    torch = _torch()
    lib = _lib.load()
    key = np.asarray(key, dtype=np.int64)
    E = int(key.size)
    if E and (key.min() < 0 or key.max() >= n):
        raise ValueError("group key out of range [0, n)")
    dkey = torch.as_tensor(key).to("cuda")
    ptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    perm = torch.zeros(max(E, 1), dtype=torch.int64, device="cuda")
    nb = lib.fcg_group_workspace_bytes(E, n)
    ws = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
    v = _lib.vp
    _lib.check(lib.fcg_group_by(v(dkey), E, n, v(ptr), v(perm), v(ws), nb, _stream(torch)),
               "fcg_group_by")
    return ptr.cpu().numpy(), perm[:E].cpu().numpy()


def group_by_destination(nl: NeighborList, n: int | None = None) -> CsrLayout:
    ptr, perm = _group(nl.dst, nl.n if n is None else n)
    return CsrLayout(ptr=ptr, perm=perm, key="dst")


def group_by_source(nl: NeighborList, n: int | None = None) -> CsrLayout:
    ptr, perm = _group(nl.src, nl.n if n is None else n)
    return CsrLayout(ptr=ptr, perm=perm, key="src")


def csr_from_neighbor_list(nl: NeighborList):
    """Convert a caller-supplied NeighborList into the device CSR form
    (ptr, nbr, rev, own).  The fused kernels need the canonical symmetric
    layout every cutoff graph has; anything else is rejected."""
    src = np.asarray(nl.src, np.int64)
    dst = np.asarray(nl.dst, np.int64)
    n, E = int(nl.n), int(src.size)
    if E:
        key = dst * n + src
        if np.any(np.diff(key) <= 0):
            raise ValueError("neighbour list must be in canonical (dst, src) order without "
                             "duplicates")
        rkey = src * n + dst
        pos_rev = np.searchsorted(key, rkey)
        if np.any(pos_rev >= E) or np.any(key[np.minimum(pos_rev, E - 1)] != rkey):
            raise ValueError("the fused GPU path needs a symmetric neighbour list "
                             "(every j->i edge paired with i->j)")
    else:
        pos_rev = np.zeros(0, np.int64)
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(dst, minlength=n), out=ptr[1:])
    return ptr, src, pos_rev, dst
