"""Structural metrics of trajectories — SURVEY §8(f) rank 4, the reference's
analysis.py surface with the per-frame work batched on the GPU.

Same names, arguments, constants and errors as flashcg.analysis
(analysis.py:1-289).  What runs where:

* kabsch_align / rmsd, fraction_native_contacts and gdt_ts evaluate on the
  GPU through libfcg (fcg_kabsch, fcg_native_q, fcg_gdt_counts, fp64); the
  ``*_batch`` variants and compute_metrics take a whole stack of frames in
  one launch each, which is where the GPU pays (GDT-TS is ~2.25 N Kabsch
  superpositions per frame, each applied to all N beads).
* graph_stats builds every frame's cutoff graph with the GPU neighbour
  builder (fcg_nbr_build, frames as replicas) and summarises the CSR.
* build_contacts (once per native structure), savitzky_golay,
  largest_metastable_q (100-bin series), read_trajectory and
  write_metrics_csv are host code.

Superposition uses Horn's quaternion form of the optimal proper rotation
(see csrc/analysis.cu); results agree with the reference's SVD to ~1e-13.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

CONTACT_BETA = 10.0          # 1/nm
CONTACT_LAMBDA = 1.5
CONTACT_CUTOFF = 0.9         # nm
CONTACT_MIN_SEPARATION = 3
GDT_CUTOFFS_NM = (0.1, 0.2, 0.4, 0.8)

Q_HIST_BINS = 100
Q_SMOOTH_WINDOW = 11
Q_SMOOTH_ORDER = 3
MIN_BASIN_DENSITY = 0.05


class DegenerateStructureError(ValueError):
    pass


@dataclass(frozen=True)
class ContactSet:
    pairs: np.ndarray       # C x 2, i < j, j - i >= separation
    ref_dist: np.ndarray    # C reference distances

    @property
    def count(self) -> int:
        return int(self.pairs.shape[0])


@dataclass
class MetricSeries:
    steps: np.ndarray
    rmsd: np.ndarray
    q: np.ndarray
    edges: np.ndarray
    gdt: np.ndarray | None = None

    def __post_init__(self):
        n = self.steps.size
        for name in ("rmsd", "q", "edges"):
            if getattr(self, name).size != n:
                raise ValueError(f"metric column {name} has mismatched length")


# ---- device plumbing ---------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_13140_b200.analysis needs a CUDA device")
    return torch


def _stream(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _frames_dev(frames, torch):
    x = np.ascontiguousarray(np.asarray(frames, dtype=np.float64))
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3 or x.shape[2] != 3:
        raise ValueError("frames must be F x N x 3")
    return x, torch.as_tensor(x).to("cuda")


def _ref_dev(x_ref, n, torch):
    y = np.ascontiguousarray(np.asarray(x_ref, dtype=np.float64))
    if y.shape != (n, 3):
        raise ValueError("structures must share an N x 3 shape")
    return torch.as_tensor(y).to("cuda")


# ---- superposition -----------------------------------------------------------

def kabsch_batch(frames, x_ref):
    """Optimal proper superposition of every frame onto x_ref (one launch).

    Returns (rot[F,3,3], trans[F,3], rmsd[F], degenerate[F] bool); moved =
    x @ rot.T + trans as in kabsch_align (analysis.py:56-81).
    """
    torch = _torch()
    x, dx = _frames_dev(frames, torch)
    F, n = x.shape[0], x.shape[1]
    dy = _ref_dev(x_ref, n, torch)
    rms = torch.empty(F, dtype=torch.float64, device="cuda")
    rot = torch.empty(F, 3, 3, dtype=torch.float64, device="cuda")
    tr = torch.empty(F, 3, dtype=torch.float64, device="cuda")
    deg = torch.empty(F, dtype=torch.int32, device="cuda")
    v = _lib.vp
    _lib.check(_lib.load().fcg_kabsch(v(dx), v(dy), F, n, v(rms), v(rot), v(tr), v(deg),
                                      _stream(torch)), "fcg_kabsch")
    return (rot.cpu().numpy(), tr.cpu().numpy(), rms.cpu().numpy(),
            deg.cpu().numpy().astype(bool))


def kabsch_align(x: np.ndarray, x_ref: np.ndarray):
    """(rotation, translation, rmsd) of the optimal proper superposition of x
    onto x_ref (analysis.py:56-81)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(x_ref, dtype=np.float64)
    if x.shape != y.shape or x.ndim != 2 or x.shape[1] != 3:
        raise ValueError("structures must share an N x 3 shape")
    if x.shape[0] < 3:
        raise DegenerateStructureError("superposition needs at least 3 beads")
    rot, tr, rms, deg = kabsch_batch(x[None], y)
    if deg[0]:
        raise DegenerateStructureError("degenerate covariance, rotation not unique")
    return rot[0], tr[0], float(rms[0])


def rmsd_batch(frames, x_ref) -> np.ndarray:
    """Kabsch RMSD of every frame against x_ref; raises on a degenerate frame."""
    frames = np.asarray(frames, dtype=np.float64)
    if frames.ndim == 3 and frames.shape[1] < 3:
        raise DegenerateStructureError("superposition needs at least 3 beads")
    _rot, _tr, rms, deg = kabsch_batch(frames, x_ref)
    if deg.any():
        raise DegenerateStructureError(
            f"degenerate covariance in frame {int(np.argmax(deg))}, rotation not unique")
    return rms


def rmsd(x: np.ndarray, x_ref: np.ndarray) -> float:
    return kabsch_align(x, x_ref)[2]


# ---- native contacts -----------------------------------------------------------

def build_contacts(x_ref: np.ndarray, cutoff: float = CONTACT_CUTOFF,
                   min_separation: int = CONTACT_MIN_SEPARATION) -> ContactSet:
    """Pairs (i, j), j - i >= min_separation, closer than cutoff in x_ref
    (analysis.py:88-97).  Host code: once per native structure."""
    x = np.asarray(x_ref, dtype=np.float64)
    i, j = np.triu_indices(x.shape[0], k=min_separation)
    dist = np.linalg.norm(x[i] - x[j], axis=1)
    sel = dist < cutoff
    return ContactSet(pairs=np.stack([i[sel], j[sel]], axis=1), ref_dist=dist[sel])


def fraction_native_contacts_batch(frames, contacts: ContactSet, beta: float = CONTACT_BETA,
                                   lam: float = CONTACT_LAMBDA) -> np.ndarray:
    """Q of every frame (one CTA per frame)."""
    if contacts.count == 0:
        raise ValueError("Q is undefined for an empty contact set")
    torch = _torch()
    x, dx = _frames_dev(frames, torch)
    F, n = x.shape[0], x.shape[1]
    pairs = torch.as_tensor(np.ascontiguousarray(contacts.pairs, dtype=np.int32)).to("cuda")
    r0 = torch.as_tensor(np.ascontiguousarray(contacts.ref_dist, dtype=np.float64)).to("cuda")
    q = torch.empty(F, dtype=torch.float64, device="cuda")
    v = _lib.vp
    _lib.check(_lib.load().fcg_native_q(v(dx), F, n, v(pairs), v(r0), contacts.count,
                                        float(beta), float(lam), v(q), _stream(torch)),
               "fcg_native_q")
    return q.cpu().numpy()


def fraction_native_contacts(x: np.ndarray, contacts: ContactSet, beta: float = CONTACT_BETA,
                             lam: float = CONTACT_LAMBDA) -> float:
    """Smooth fraction of preserved contacts in [0, 1] (analysis.py:100-108)."""
    return float(fraction_native_contacts_batch(np.asarray(x)[None], contacts, beta, lam)[0])


# ---- GDT-TS -------------------------------------------------------------------

def gdt_windows(n: int) -> np.ndarray:
    """Seed windows (start, length) of the GDT-TS search: every contiguous
    window of length n, n/2 and n/4 (at least 3), longest first
    (analysis.py:111-131)."""
    out = []
    for length in sorted({n, max(n // 2, 3), max(n // 4, 3)}, reverse=True):
        out.extend((s, length) for s in range(0, n - length + 1))
    return np.asarray(out, dtype=np.int32).reshape(-1, 2)


def gdt_ts_batch(frames, x_ref) -> np.ndarray:
    """GDT-TS of every frame against x_ref: all seeds of all frames in one
    launch, best count per cutoff on the device, mean of count / N here."""
    torch = _torch()
    x, dx = _frames_dev(frames, torch)
    F, n = x.shape[0], x.shape[1]
    if n < 3:
        raise DegenerateStructureError("GDT-TS needs at least 3 beads")
    dy = _ref_dev(x_ref, n, torch)
    win = gdt_windows(n)
    dwin = torch.as_tensor(np.ascontiguousarray(win)).to("cuda")
    cut = (C.c_double * 4)(*GDT_CUTOFFS_NM)
    best = torch.empty(F, 4, dtype=torch.int32, device="cuda")
    v = _lib.vp
    _lib.check(_lib.load().fcg_gdt_counts(v(dx), v(dy), F, n, v(dwin), int(win.shape[0]),
                                          C.cast(cut, C.c_void_p), v(best), _stream(torch)),
               "fcg_gdt_counts")
    frac = best.cpu().numpy().astype(np.int64) / n
    return np.array([float(row.mean()) for row in frac])


def gdt_ts(x: np.ndarray, x_ref: np.ndarray) -> float:
    """Cutoff-ladder similarity with the multi-seed superposition search
    (analysis.py:115-143)."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[0] < 3:
        raise DegenerateStructureError("GDT-TS needs at least 3 beads")
    return float(gdt_ts_batch(x[None], x_ref)[0])


# ---- series analysis (host) ----------------------------------------------------

def savitzky_golay(series: np.ndarray, window: int, order: int) -> np.ndarray:
    """Local least-squares polynomial smoothing; the ends are evaluated from
    one polynomial fitted to the first (last) window (analysis.py:146-176)."""
    y = np.asarray(series, dtype=np.float64)
    if window % 2 != 1 or window <= order:
        raise ValueError("window must be odd and larger than order")
    if y.ndim != 1 or y.size < window:
        raise ValueError("series must be 1-d with at least window entries")
    half = window // 2
    # least-squares fit over offsets -half..half; the smoothed value is the
    # fitted constant term, a fixed linear combination of the window
    t = np.arange(-half, half + 1, dtype=np.float64)
    design = t[:, None] ** np.arange(order + 1)[None, :]
    center_row = np.linalg.pinv(design)[0]
    out = np.empty_like(y)
    out[half:y.size - half] = np.lib.stride_tricks.sliding_window_view(y, window) @ center_row
    pos = np.arange(window, dtype=np.float64)
    basis = pos[:, None] ** np.arange(order + 1)[None, :]
    for seg, sl_out, sl_fit in ((y[:window], slice(0, half), slice(0, half)),
                                (y[-window:], slice(y.size - half, y.size),
                                 slice(window - half, window))):
        coef = np.linalg.lstsq(basis, seg, rcond=None)[0]
        out[sl_out] = (basis @ coef)[sl_fit]
    return out


def largest_metastable_q(q_series: np.ndarray, bins: int = Q_HIST_BINS,
                         window: int = Q_SMOOTH_WINDOW, order: int = Q_SMOOTH_ORDER) -> float:
    """Q of the rightmost basin of the smoothed Q density: the last strict
    interior local maximum reaching MIN_BASIN_DENSITY of the peak, else the
    global maximum (analysis.py:179-205)."""
    q = np.asarray(q_series, dtype=np.float64)
    if q.size == 0:
        raise ValueError("empty Q series")
    if np.ptp(q) == 0.0:
        return float(q[0])
    density, edges = np.histogram(q, bins=bins, range=(0.0, 1.0), density=True)
    sm = savitzky_golay(density, window, order)
    centers = 0.5 * (edges[:-1] + edges[1:])
    floor = MIN_BASIN_DENSITY * float(sm.max())
    peak = (sm[1:-1] > sm[:-2]) & (sm[1:-1] > sm[2:]) & (sm[1:-1] >= floor)
    idx = np.flatnonzero(peak)
    return float(centers[idx[-1] + 1] if idx.size else centers[int(np.argmax(sm))])


# ---- graph statistics (GPU neighbour build) -------------------------------------

def graph_stats(frames, r_cut: float):
    """Per-frame E, mean/max degree and mean/max sequence separation of the
    cutoff graph (analysis.py:208-231), all frames built in one
    fcg_nbr_build call (frames as replicas)."""
    x = np.asarray([np.asarray(f) for f in frames])
    if x.ndim != 3 or x.shape[2] != 3:
        raise ValueError("frames must share an N x 3 shape")
    # the builder sizes its edge buffers for the dense worst case F*N*(N-1):
    # batch the frames so that stays ~64M slots
    step = max(1, (64 << 20) // max(x.shape[1] * max(x.shape[1] - 1, 1), 1))
    parts = [_graph_stats_batch(x[a:a + step], r_cut) for a in range(0, x.shape[0], step)]
    return {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}


def _graph_stats_batch(x, r_cut):
    from .csr import device_csr
    F, n = x.shape[0], x.shape[1]
    ptr, nbr, _rev, own = device_csr(x, r_cut)
    starts = ptr[0:F * n:n]
    edges = ptr[n::n][:F] - starts
    deg = np.diff(ptr).reshape(F, n)
    E = int(ptr[-1])
    span = np.abs(own[:E] - nbr[:E])
    frame_of = np.repeat(np.arange(F), edges)
    with np.errstate(invalid="ignore", divide="ignore"):
        span_sum = np.bincount(frame_of, weights=span, minlength=F)
        mean_span = np.where(edges > 0, span_sum / np.maximum(edges, 1), 0.0)
    max_span = np.zeros(F, dtype=np.int64)
    if E:
        np.maximum.at(max_span, frame_of, span)
    return {
        "edges": edges.astype(np.int64),
        "mean_degree": np.where(edges > 0, deg.mean(axis=1), 0.0),
        "max_degree": np.where(edges > 0, deg.max(axis=1), 0).astype(np.int64),
        "mean_span": mean_span,
        "max_span": max_span,
    }


# ---- trajectories and metric files ------------------------------------------------

def read_trajectory(path):
    """Frames (step, replica, types, positions) of an XYZ trajectory written
    by run_simulation (analysis.py:234-257)."""
    with open(path) as fh:
        lines = fh.read().splitlines()
    frames, i = [], 0
    while i < len(lines):
        if not lines[i].strip():
            i += 1
            continue
        n = int(lines[i])
        meta = dict(kv.split("=") for kv in lines[i + 1].split())
        rows = [ln.split() for ln in lines[i + 2:i + 2 + n]]
        types = np.array([int(r[0].lstrip("B")) for r in rows])
        coords = np.array([[float(v) for v in r[1:4]] for r in rows])
        frames.append((int(meta["step"]), int(meta["replica"]), types, coords))
        i += 2 + n
    if not frames:
        raise ValueError(f"{path}: empty trajectory")
    return frames


def compute_metrics(frames, native: np.ndarray, r_cut: float,
                    contacts: ContactSet | None = None, with_gdt: bool = False) -> MetricSeries:
    """Per-frame RMSD, Q, edge count (and GDT-TS) against the native
    structure (analysis.py:260-276), each metric one batched GPU launch."""
    if contacts is None:
        contacts = build_contacts(native)
    steps = np.array([f[0] for f in frames])
    pos = np.asarray([np.asarray(f[3], dtype=np.float64) for f in frames])
    return MetricSeries(steps=steps, rmsd=rmsd_batch(pos, native),
                        q=fraction_native_contacts_batch(pos, contacts),
                        edges=graph_stats(pos, r_cut)["edges"],
                        gdt=gdt_ts_batch(pos, native) if with_gdt else None)


def write_metrics_csv(series: MetricSeries, path) -> None:
    """flashcg-metrics v1 CSV (analysis.py:279-289)."""
    cols = ["frame", "step", "rmsd", "q", "edges"] + (["gdt_ts"] if series.gdt is not None else [])
    out = ["# flashcg-metrics v1", ",".join(cols)]
    for k in range(series.steps.size):
        row = [str(k), str(series.steps[k]), f"{series.rmsd[k]:.8f}", f"{series.q[k]:.8f}",
               str(series.edges[k])]
        if series.gdt is not None:
            row.append(f"{series.gdt[k]:.8f}")
        out.append(",".join(row))
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")
