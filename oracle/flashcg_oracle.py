"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference's per-step MD path (flashcg, read from
/root/reference/pkg/src/flashcg) used as the checker by tests/, by
__graft_entry__.smoke() and by the CPU-baseline leg of bench.py.  Nothing in
the package paper_2602_13140_b200 imports this module.

Pinning: tests/test_oracle_golden.py compares every function here against
golden vectors produced by running the reference itself
(tests/golden/make_golden.py, committed with its outputs): bit-exact for
the neighbour list / CSR / noise / one integrator step, within fp32
round-off (1e-6 relative) for energies and forces.

Third-party arithmetic the reference relies on (numpy 2.3.5 here): the
fp64 einsum association, reduceat, Philox-4x64-10 + the ziggurat normal
sampler.  The noise below calls numpy's own Generator(Philox), i.e. the
same third-party implementation the reference calls (md.py:127-131).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

KB = 0.00831446261815324          # md.py:29
FORCE_BLOWUP_LIMIT = 1.0e6         # md.py:30
TINY_DISTANCE = 1e-12              # reference.py:36
LN2 = math.log(2.0)                # model.py:16


# ---------------------------------------------------------------------------
# (a) neighbour list + CSR  (neighbors.py:47-132)

def neighbor_list(positions, r_cut, chunk=512):
    """Edges (j -> i) with fp64 dist2 < r_cut*r_cut, i != j, canonical
    (dst, src) order.  dist2 is formed as (dx*dx + dz*dz) + dy*dy, the
    association numpy's einsum("ijk,ijk->ij") uses in the reference
    (neighbors.py:59-61, :96-98)."""
    r = np.asarray(positions, dtype=np.float64)
    n = r.shape[0]
    if n == 0:
        raise ValueError("need at least one bead")
    cut2 = r_cut * r_cut
    dsts, srcs = [], []
    for a in range(0, n, chunk):
        blk = r[a:a + chunk]
        dx = blk[:, None, 0] - r[None, :, 0]
        dy = blk[:, None, 1] - r[None, :, 1]
        dz = blk[:, None, 2] - r[None, :, 2]
        d2 = (dx * dx + dz * dz) + dy * dy
        mask = d2 < cut2
        rows = np.arange(a, a + blk.shape[0])
        mask[rows - a, rows] = False
        di, sj = np.nonzero(mask)           # row-major == (dst, src) order
        dsts.append(di + a)
        srcs.append(sj)
    return np.concatenate(srcs).astype(np.int64), np.concatenate(dsts).astype(np.int64)


def group(key, n):
    """(ptr, perm): exclusive cumsum of bincount and a stable argsort
    (neighbors.py:113-120)."""
    key = np.asarray(key, dtype=np.int64)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(key, minlength=n), out=ptr[1:])
    return ptr, np.argsort(key, kind="stable").astype(np.int64)


def segment_sum(values, ptr):
    """Sum rows of each CSR segment; empty segments give zero rows
    (flash.py:109-135 without the >split chunking, which only changes
    rounding order)."""
    values = np.asarray(values)
    out = np.zeros((ptr.size - 1,) + values.shape[1:], dtype=values.dtype)
    sizes = np.diff(ptr)
    live = sizes > 0
    if values.shape[0] and np.any(live):
        out[live] = np.add.reduceat(values, ptr[:-1][live], axis=0)
    return out


# ---------------------------------------------------------------------------
# (b) model primitives  (model.py:93-157)

def ssp(x):
    return np.maximum(x, 0) + np.log1p(np.exp(-np.abs(x))) - x.dtype.type(LN2)


def ssp_grad(x):
    h = x.dtype.type(0.5)
    return h * (1.0 + np.tanh(h * x))


def _envelope(d, cutoff):
    inside = d < cutoff
    c = np.where(inside, 0.5 * (np.cos(np.pi * d / cutoff) + 1.0), 0.0).astype(d.dtype, copy=False)
    dc = np.where(inside, -0.5 * np.pi / cutoff * np.sin(np.pi * d / cutoff), 0.0
                  ).astype(d.dtype, copy=False)
    return c, dc


def basis(d, rbf, with_grad=False):
    """Enveloped Gaussian basis b[e,k] = exp(-g*(d-mu_k)^2)*C(d) and, if asked,
    db/dd = g_k*(-2*g*(d-mu_k)*C + C')  (model.py:123-157)."""
    mu = np.asarray(rbf.centers).astype(d.dtype, copy=False)
    g = d.dtype.type(rbf.gamma)
    delta = d[:, None] - mu
    gauss = np.exp(-g * delta * delta)
    c, dc = _envelope(d, rbf.cutoff)
    b = gauss * c[:, None]
    if not with_grad:
        return b
    return b, gauss * (-2.0 * g * delta * c[:, None] + dc[:, None])


# ---------------------------------------------------------------------------
# linear layers: plain (W, b) tuples or quantized modules (quantize.py:55-98)

def _layers(net):
    return net if isinstance(net, tuple) else net.layers


def _lin_fwd(lin, x):
    if isinstance(lin, tuple):
        return x @ lin[0].T + lin[1]
    x16 = x.astype(np.float16).astype(np.float32)          # quantize.py:68-71
    w = lin.scale[:, None] * lin.weight.astype(np.float32)
    return x16 @ w.T + lin.bias


def _lin_mat(lin):
    return lin[0] if isinstance(lin, tuple) else lin.scale[:, None] * lin.weight.astype(np.float32)


def mlp_fwd(net, x):
    """Returns (out, preacts); ssp after every layer but the last, hidden
    activations rounded to fp16 for quantized nets (quantize.py:80-88)."""
    quant = not isinstance(net, tuple)
    layers = _layers(net)
    pre, a = [], x
    for i, lin in enumerate(layers):
        z = _lin_fwd(lin, a)
        if i < len(layers) - 1:
            pre.append(z)
            a = ssp(z)
            if quant:
                a = a.astype(np.float16).astype(np.float32)
        else:
            a = z
    return a, pre


def mlp_bwd(net, pre, g):
    layers = _layers(net)
    for i in range(len(layers) - 1, -1, -1):
        g = g @ _lin_mat(layers[i])
        if i > 0:
            g = g * ssp_grad(pre[i - 1])
    return g


# ---------------------------------------------------------------------------
# (b)(c)(d) fused-flash restatement: dst-grouped forward, src-grouped
# backward, segment sums instead of scatters (flash.py:192-307, :446-501)

def energy_forces(positions, types, params, edges=None):
    """Returns (energy, per_atom, forces) like flash_energy_forces."""
    pos = np.asarray(positions)
    types = np.asarray(types)
    cfg = params.config
    if np.any(types < 0) or np.any(types >= cfg.num_atom_types):
        raise ValueError("atom type out of range for the embedding table")
    n = pos.shape[0]
    src, dst = edges if edges is not None else neighbor_list(pos, cfg.cutoff)
    dptr, dperm = group(dst, n)
    sptr, sperm = group(src, n)
    dt = pos.dtype

    u = pos[dst] - pos[src]
    d = np.sqrt(u[:, 0] * u[:, 0] + u[:, 1] * u[:, 1] + u[:, 2] * u[:, 2])
    safe = d > TINY_DISTANCE
    inv_d = np.where(safe, 1.0 / np.where(safe, d, 1.0), 0.0).astype(dt, copy=False)

    X = params.embedding[types].astype(dt, copy=False)
    saved = []
    for bp in params.blocks:
        P = _lin_fwd(bp.pre_linear, X)
        b = basis(d, params.rbf)
        w, _ = mlp_fwd(bp.filter_mlp, b)
        H = segment_sum((P[src] * w)[dperm], dptr)
        U, post_pre = mlp_fwd(bp.post_mlp, H)
        saved.append((P, post_pre))
        X = X + U

    eps, ro_pre = mlp_fwd(params.readout, X)
    per_atom = eps[:, 0]
    energy = float(per_atom.sum())

    G = mlp_bwd(params.readout, ro_pre, np.ones((n, 1), dtype=dt))
    grad_r = np.zeros((n, 3), dtype=dt)
    for (P, post_pre), bp in zip(reversed(saved), reversed(params.blocks)):
        GH = mlp_bwd(bp.post_mlp, post_pre, G)
        b, db = basis(d, params.rbf, with_grad=True)
        w, fpre = mlp_fwd(bp.filter_mlp, b)
        gH = GH[dst]
        GP = segment_sum((gH * w)[sperm], sptr)
        gb = mlp_bwd(bp.filter_mlp, fpre, gH * P[src])
        gd = np.einsum("ek,ek->e", gb, db)
        g = (gd * inv_d)[:, None] * u
        grad_r += segment_sum(g[dperm], dptr) - segment_sum(g[sperm], sptr)
        G = G + GP @ _lin_mat(bp.pre_linear)
    return energy, per_atom, -grad_r


# ---------------------------------------------------------------------------
# (f) integrator  (md.py:109-185)

def prior_energy_forces(positions, prior):
    if prior is None or prior.num_bonds == 0:
        return 0.0, np.zeros_like(positions)
    i, j = prior.bonds[:, 0], prior.bonds[:, 1]
    rij = positions[i] - positions[j]
    d = np.sqrt(rij[:, 0] * rij[:, 0] + rij[:, 1] * rij[:, 1] + rij[:, 2] * rij[:, 2])
    st = d - prior.rest_length.astype(positions.dtype)
    k = prior.spring_k.astype(positions.dtype)
    energy = float(0.5 * np.sum(k * st * st))
    f = (-k * st / np.where(d > 0, d, 1.0))[:, None] * rij
    out = np.zeros_like(positions)
    np.add.at(out, i, f)
    np.add.at(out, j, -f)
    return energy, out


def noise(seed, replica, step, n, dtype=np.float32):
    g = np.random.Generator(np.random.Philox(key=np.array([seed, replica], dtype=np.uint64),
                                             counter=np.array([0, 0, 0, step], dtype=np.uint64)))
    return g.standard_normal((n, 3)).astype(dtype)


def coefficients(dt_fs, temperature, friction):
    dt = dt_fs * 1e-3
    c1 = math.exp(-friction * dt)
    return 0.5 * dt, c1, (1.0 - c1 * c1) * KB * temperature


def baoa(pos, vel, forces, masses, xi, dt_fs, temperature, friction):
    """langevin_step without the trailing kick (md.py:158-172); numpy applies
    the NEP 50 fp32 rounding of the Python-float coefficients."""
    h, c1, c2n = coefficients(dt_fs, temperature, friction)
    m = masses[None, :, None].astype(vel.dtype)
    v = vel + h * forces / m
    r = pos + h * v
    v = c1 * v + np.sqrt(c2n / m) * xi
    r = r + h * v
    return r, v


def half_kick(vel, forces, masses, dt_fs):
    m = masses[None, :, None].astype(vel.dtype)
    return vel + (0.5 * dt_fs * 1e-3) * forces / m


def kinetic_temperature(vel, masses):
    m = masses[None, :, None]
    ke = 0.5 * np.sum(m * vel ** 2, axis=(1, 2))
    return 2.0 * ke / (3 * vel.shape[1] * KB)


def replica_forces(params, types, prior, positions, workers=1, edges=None):
    """Per-replica model + prior forces (md.py:243-273); `edges` optionally
    gives a cached (src, dst) per replica (neighbor_stride > 1)."""
    def one(rep):
        e, _, f = energy_forces(positions[rep], types, params,
                                edges=None if edges is None else edges[rep])
        ep, fp = prior_energy_forces(positions[rep], prior)
        return e, ep, f + fp
    reps = range(positions.shape[0])
    if workers > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(one, reps))
    else:
        res = [one(r) for r in reps]
    forces = np.stack([r[2] for r in res]).astype(positions.dtype)
    return forces, np.array([r[0] for r in res]), np.array([r[1] for r in res])


def run_md(params, types, masses, prior, positions, velocities, n_steps, dt_fs=4.0,
           temperature=300.0, friction=1.0, seed=0, step0=0, rep_offset=0, workers=1,
           record=False, neighbor_stride=1):
    """BAOAB loop with one force evaluation per step (md.py:188-208).
    Returns (positions, velocities, forces, potential, prior, trace)."""
    pos = np.array(positions, dtype=np.float32)
    vel = np.array(velocities, dtype=np.float32)
    R, N = pos.shape[0], pos.shape[1]
    cut = params.config.cutoff
    cache = [neighbor_list(pos[r], cut) for r in range(R)]
    F, pot, pri = replica_forces(params, types, prior, pos, workers, edges=cache)
    trace = [(step0, pot, pri)] if record else None
    step = step0
    for _ in range(n_steps):
        xi = np.stack([noise(seed, rep_offset + r, step, N) for r in range(R)])
        pos, vel = baoa(pos, vel, F, masses, xi, dt_fs, temperature, friction)
        step += 1
        if step % max(neighbor_stride, 1) == 0:  # md.py:245-250
            cache = [neighbor_list(pos[r], cut) for r in range(R)]
        F, pot, pri = replica_forces(params, types, prior, pos, workers, edges=cache)
        vel = half_kick(vel, F, masses, dt_fs)
        if record:
            trace.append((step, pot, pri))
    return pos, vel, F, pot, pri, trace


# ---------------------------------------------------------------------------
# parity metrics (verify.py:62-74)

def energy_rel_err(e_test, e_ref, per_atom_ref):
    scale = max(abs(e_ref), float(np.linalg.norm(per_atom_ref)), 1e-300)
    return abs(e_test - e_ref) / scale


def force_rel_err(f_test, f_ref):
    scale = float(np.max(np.linalg.norm(f_ref, axis=-1))) + 1e-300
    return float(np.max(np.linalg.norm(f_test - f_ref, axis=-1))) / scale
