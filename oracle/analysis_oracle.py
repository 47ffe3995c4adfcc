"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference's trajectory analysis
(/root/reference/pkg/src/flashcg/analysis.py), the checker for the GPU
analysis module (paper_2602_13140_b200/analysis.py, csrc/analysis.cu).
Only tests/ import it.

Pinning: tests/test_analysis.py compares every function here with golden
vectors produced by running the reference itself
(tests/golden/make_analysis_golden.py -> tests/golden/analysis.npz).
Third-party arithmetic: numpy's LAPACK SVD (dgesdd) in the Kabsch step and
numpy's pairwise means; the oracle calls the same numpy routines.
"""

from __future__ import annotations

import numpy as np

CONTACT_BETA = 10.0          # analysis.py:16
CONTACT_LAMBDA = 1.5         # analysis.py:17
CONTACT_CUTOFF = 0.9         # analysis.py:18
CONTACT_MIN_SEPARATION = 3   # analysis.py:19
GDT_CUTOFFS_NM = (0.1, 0.2, 0.4, 0.8)  # analysis.py:20


class Degenerate(ValueError):
    pass


def kabsch(x, y):
    """analysis.py:56-81: SVD of xc^T yc, proper rotation V diag(1,1,d) U^T."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if x.shape[0] < 3:
        raise Degenerate("fewer than 3 beads")
    xm, ym = x.mean(axis=0), y.mean(axis=0)
    xc, yc = x - xm, y - ym
    u, s, vt = np.linalg.svd(xc.T @ yc)
    if s[1] <= 1e-12 * max(s[0], 1.0):
        raise Degenerate("degenerate covariance")
    d = np.sign(np.linalg.det(vt.T @ u.T))
    rot = vt.T @ np.diag([1.0, 1.0, d]) @ u.T
    moved = xc @ rot.T
    return rot, ym - rot @ xm, float(np.sqrt(np.mean(np.sum((moved - yc) ** 2, axis=1))))


def contacts(x_ref, cutoff=CONTACT_CUTOFF, min_separation=CONTACT_MIN_SEPARATION):
    """analysis.py:88-97."""
    x = np.asarray(x_ref, np.float64)
    ii, jj = np.triu_indices(x.shape[0], k=min_separation)
    d = np.linalg.norm(x[ii] - x[jj], axis=1)
    keep = d < cutoff
    return np.stack([ii[keep], jj[keep]], axis=1), d[keep]


def native_q(x, pairs, ref_dist, beta=CONTACT_BETA, lam=CONTACT_LAMBDA):
    """analysis.py:100-108."""
    x = np.asarray(x, np.float64)
    r = np.linalg.norm(x[pairs[:, 0]] - x[pairs[:, 1]], axis=1)
    return float(np.mean(1.0 / (1.0 + np.exp(beta * (r - lam * ref_dist)))))


def gdt_best_counts(x, y):
    """analysis.py:115-143 as integer counts: best number of beads within each
    cutoff over all non-degenerate seeds (GDT-TS = mean(counts / n))."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    n = x.shape[0]
    best = np.zeros(len(GDT_CUTOFFS_NM), dtype=np.int64)
    for length in sorted({n, max(n // 2, 3), max(n // 4, 3)}, reverse=True):
        for start in range(0, n - length + 1):
            try:
                rot, trans, _ = kabsch(x[start:start + length], y[start:start + length])
            except Degenerate:
                continue
            dist = np.linalg.norm(x @ rot.T + trans - y, axis=1)
            for c, cut in enumerate(GDT_CUTOFFS_NM):
                best[c] = max(best[c], int(np.count_nonzero(dist <= cut)))
    return best


def gdt_ts(x, y):
    return float((gdt_best_counts(x, y) / np.asarray(x).shape[0]).mean())


def savgol(y, window, order):
    """analysis.py:146-176."""
    y = np.asarray(y, np.float64)
    half = window // 2
    a = np.vander(np.arange(-half, half + 1, dtype=np.float64), order + 1, increasing=True)
    out = np.empty_like(y)
    out[half:-half] = np.convolve(y, np.linalg.pinv(a)[0][::-1], mode="valid")
    basis = np.vander(np.arange(window, dtype=np.float64), order + 1, increasing=True)
    out[:half] = (basis @ np.linalg.lstsq(basis, y[:window], rcond=None)[0])[:half]
    out[-half:] = (basis @ np.linalg.lstsq(basis, y[-window:], rcond=None)[0])[-half:]
    return out


def largest_metastable_q(q, bins=100, window=11, order=3, floor_frac=0.05):
    """analysis.py:179-205."""
    q = np.asarray(q, np.float64)
    if np.ptp(q) == 0.0:
        return float(q[0])
    dens, edges = np.histogram(q, bins=bins, range=(0.0, 1.0), density=True)
    sm = savgol(dens, window, order)
    centers = 0.5 * (edges[:-1] + edges[1:])
    mid = sm[1:-1]
    idx = np.nonzero((mid > sm[:-2]) & (mid > sm[2:]) & (mid >= floor_frac * sm.max()))[0]
    return float(centers[idx[-1] + 1] if idx.size else centers[int(np.argmax(sm))])


def graph_stats(frames, r_cut):
    """analysis.py:208-231 over the brute-force fp64 cutoff graph."""
    from .flashcg_oracle import neighbor_list
    rows = []
    for pos in frames:
        src, dst = neighbor_list(pos, r_cut)
        n = np.asarray(pos).shape[0]
        if src.size:
            deg = np.bincount(dst, minlength=n)
            span = np.abs(src - dst)
            rows.append((src.size, float(deg.mean()), int(deg.max()), float(span.mean()),
                         int(span.max())))
        else:
            rows.append((0, 0.0, 0, 0.0, 0))
    a = np.array(rows, dtype=np.float64)
    return {"edges": a[:, 0].astype(np.int64), "mean_degree": a[:, 1],
            "max_degree": a[:, 2].astype(np.int64), "mean_span": a[:, 3],
            "max_span": a[:, 4].astype(np.int64)}
