"""FLCG checkpoint container (kind 1), compatible with the reference's
params_io.save_checkpoint / load_checkpoint (params_io.py:206-233).

Layout (little-endian): b"FLCG" | u32 version=1 | u32 kind=1 |
u64 step | u64 seed | u32 replicas | u32 beads | u32 tensor count, then per
tensor: u16 name length | name | u8 tag (0 fp32, 1 fp64) | u8 rank |
u32 dims[rank] | row-major payload.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"FLCG"
VERSION = 1
KIND_CHECKPOINT = 1


class FileFormatError(ValueError):
    pass


def _put(f, name: str, arr: np.ndarray):
    arr = np.asarray(arr)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float32)
    tag = 1 if arr.dtype == np.float64 else 0
    b = name.encode()
    f.write(struct.pack("<H", len(b)) + b + struct.pack("<BB", tag, arr.ndim))
    f.write(struct.pack(f"<{arr.ndim}I", *arr.shape))
    f.write(np.ascontiguousarray(arr).astype("<f8" if tag else "<f4").tobytes())


def _take(f, n, what):
    b = f.read(n)
    if len(b) != n:
        raise FileFormatError(f"truncated file while reading {what}")
    return b


def _get(f):
    (ln,) = struct.unpack("<H", _take(f, 2, "name length"))
    name = _take(f, ln, "name").decode()
    tag, rank = struct.unpack("<BB", _take(f, 2, f"header of {name}"))
    if tag not in (0, 1):
        raise FileFormatError(f"unsupported precision tag {tag} on tensor {name}")
    dims = struct.unpack(f"<{rank}I", _take(f, 4 * rank, f"dims of {name}"))
    dt = np.dtype("<f8" if tag else "<f4")
    n = int(np.prod(dims, dtype=np.int64)) if rank else 1
    arr = np.frombuffer(_take(f, n * dt.itemsize, f"payload of {name}"), dtype=dt)
    return name, arr.reshape(dims).astype(np.float64 if tag else np.float32)


def save_checkpoint(path, positions, velocities, masses, step: int, seed: int) -> None:
    positions = np.asarray(positions)
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<II", VERSION, KIND_CHECKPOINT))
        f.write(struct.pack("<QQII", int(step), int(seed), positions.shape[0], positions.shape[1]))
        f.write(struct.pack("<I", 3))
        _put(f, "positions", positions)
        _put(f, "velocities", velocities)
        _put(f, "masses", masses)


def load_checkpoint(path) -> dict:
    with open(path, "rb") as f:
        if _take(f, 4, "magic") != MAGIC:
            raise FileFormatError(f"{path}: not an FLCG file")
        version, kind = struct.unpack("<II", _take(f, 8, "header"))
        if version != VERSION or kind != KIND_CHECKPOINT:
            raise FileFormatError(f"{path}: expected a version-1 checkpoint")
        step, seed, n_rep, n_beads = struct.unpack("<QQII", _take(f, 24, "checkpoint header"))
        (count,) = struct.unpack("<I", _take(f, 4, "tensor count"))
        out = dict(_get(f) for _ in range(count))
    for k in ("positions", "velocities", "masses"):
        if k not in out:
            raise FileFormatError(f"missing tensor {k}")
    if out["positions"].shape[:2] != (n_rep, n_beads):
        raise FileFormatError("tensor positions does not match the checkpoint header")
    return {"step": step, "seed": seed, **out}
