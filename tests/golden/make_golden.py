"""Generate the golden fixtures by running the REFERENCE (flashcg) itself.

Run here, where /root/reference exists (it does not on the GPU box):
    python tests/golden/make_golden.py
Outputs tests/golden/*.npz and hashes.json (committed).  The fixtures pin
the CPU oracle (oracle/flashcg_oracle.py) and the host-side input
generators; GPU tests compare the CUDA path against the oracle and these.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from flashcg import flash as RF  # noqa: E402
from flashcg import md as RMD  # noqa: E402
from flashcg import model as RM  # noqa: E402
from flashcg import neighbors as RN  # noqa: E402
from flashcg import quantize as RQ  # noqa: E402
from flashcg import reference as RR  # noqa: E402
from flashcg import systems as RS  # noqa: E402

SMALL = dict(hidden_dim=16, rbf_dim=8, num_blocks=2, cutoff=1.0, num_atom_types=6,
             filter_hidden_dim=16, readout_hidden_dim=8)
TINY = dict(hidden_dim=8, rbf_dim=4, num_blocks=1, cutoff=1.2, num_atom_types=8,
            filter_hidden_dim=8, readout_hidden_dim=4)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def params_hash(p) -> str:
    h = hashlib.sha256()
    for name, arr in p.named_tensors():
        h.update(name.encode())
        h.update(sha(arr).encode())
    return h.hexdigest()


def neighbors_fixture():
    cases = {}

    def add(name, pos, rc):
        pos = np.asarray(pos)
        nl = RN.build_neighbors_cells(pos, rc)
        bf = RN.build_neighbors_bruteforce(pos, rc)
        assert np.array_equal(nl.src, bf.src) and np.array_equal(nl.dst, bf.dst)
        d, s = RN.group_by_destination(nl), RN.group_by_source(nl)
        cases[name] = dict(pos=pos, rc=np.float64(rc), src=nl.src, dst=nl.dst, dptr=d.ptr,
                           dperm=d.perm, sptr=s.ptr, sperm=s.perm)

    # known-answer cases of tests/test_neighbors.py:15-48
    add("two_beads", [[0.0, 0, 0], [0.5, 0, 0]], 1.0)
    add("cutoff_strict", [[0.0, 0, 0], [1.0, 0, 0]], 1.0)
    add("single", np.zeros((1, 3)), 1.0)
    line = np.zeros((6, 3))
    line[:, 0] = np.arange(6) * 2.0
    add("spread_line", line, 1.0)
    add("triangle", [[0.0, 0, 0], [0.4, 0, 0], [0.2, 0.3, 0]], 1.0)
    add("coincident", np.zeros((4, 3)), 1.0)
    # randomized, both geometries of tests/test_neighbors.py:51-65 / verify.py:97-116
    rng = np.random.default_rng(11)
    for t in range(24):
        n = int(rng.integers(1, 300))
        if t % 3 == 0:
            c = rng.uniform(0, 5.0, size=(max(n // 20, 1), 3))
            pos = c[rng.integers(0, c.shape[0], n)] + rng.normal(0, 0.25, size=(n, 3))
        else:
            pos = rng.uniform(0, rng.uniform(0.5, 3.0) * n ** (1 / 3), size=(n, 3))
        if t % 2:
            pos = pos.astype(np.float32)
        add(f"random{t}", pos, float(rng.uniform(0.4, 1.6)))
    sysm = RS.generate_system("coil", 269, 0)
    add("coil269_f32", sysm.positions.astype(np.float32), 1.5)
    # adversarial fp64 pairs whose dist2 sits within an ulp of r_cut^2, where
    # the association of the 3-term sum decides the edge
    rng = np.random.default_rng(1)
    pairs = []
    rc = 1.5
    while len(pairs) < 256:
        a = rng.uniform(0, 2, size=(200000, 3))
        u = rng.normal(size=(200000, 3))
        u /= np.linalg.norm(u, axis=1)[:, None]
        b = a + u * rc * (1 + rng.normal(size=(200000, 1)) * 1e-16)
        dx, dy, dz = (a - b).T
        s1 = (dx * dx + dz * dz) + dy * dy
        s2 = (dx * dx + dy * dy) + dz * dz
        for k in np.nonzero((s1 < rc * rc) != (s2 < rc * rc))[0][:64]:
            pairs.append(np.stack([a[k], b[k]]))
    pairs = np.stack(pairs[:256])
    edge = np.array([RN.build_neighbors_cells(p, rc).num_edges > 0 for p in pairs])
    flat = {}
    for name, c in cases.items():
        for k, v in c.items():
            flat[f"{name}/{k}"] = v
    flat["adversarial/pairs"] = pairs
    flat["adversarial/rc"] = np.float64(rc)
    flat["adversarial/edge"] = edge
    np.savez_compressed(OUT / "neighbors.npz", **flat)


def flash_fixture():
    out = {}

    def add(name, pos, types, cfg, pseed, dtype=np.float32, nl=None, quant=False):
        params = RM.init_params(RM.ModelConfig(**cfg), pseed)
        if dtype == np.float64:
            params = params.astype(np.float64)
        if quant:
            params = RQ.quantize_model(params, seed=0)
        fl = RF.flash_energy_forces(pos, types, params, RF.PipelineMode(), nl=nl)
        ref = RR.reference_energy_forces(pos, types, params, nl=nl)
        out.update({f"{name}/pos": pos, f"{name}/types": types, f"{name}/pseed": pseed,
                    f"{name}/cfg": json.dumps(cfg), f"{name}/quant": quant,
                    f"{name}/energy": fl.energy, f"{name}/per_atom": fl.per_atom,
                    f"{name}/forces": fl.forces, f"{name}/ref_energy": ref.energy,
                    f"{name}/ref_forces": ref.forces,
                    f"{name}/traffic_total": fl.traffic.total_bytes})

    for seed in range(4):   # tests/test_flash.py:26-33 instances
        rng = np.random.default_rng(seed)
        pos = rng.uniform(0, 1.6, size=(24, 3)).astype(np.float32)
        add(f"small{seed}", pos, rng.integers(0, 6, size=24), SMALL, seed)
    rng = np.random.default_rng(5)
    pos = rng.uniform(0, 1.6, size=(24, 3))
    add("small64", pos, rng.integers(0, 6, size=24), SMALL, 5, dtype=np.float64)
    star = np.zeros((7, 3), dtype=np.float32)
    star[1:] = 0.95 * np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1],
                                [0, 0, -1]], dtype=np.float32)
    add("star", star, np.random.default_rng(2).integers(0, 6, size=7), SMALL, 2)
    rng = np.random.default_rng(1)
    spread = (rng.uniform(0, 1.6, size=(5, 3)) + np.arange(5)[:, None] * 50.0).astype(np.float32)
    add("no_edges", spread, rng.integers(0, 6, size=5), SMALL, 1)
    full = dict(hidden_dim=128, rbf_dim=64, num_blocks=3, cutoff=1.5, num_atom_types=32,
                filter_hidden_dim=128, readout_hidden_dim=64)
    sysm = RS.generate_system("coil", 269, 0)
    add("coil269", sysm.positions.astype(np.float32), sysm.types, full, 0)
    glob = RS.generate_system("globule", 269, 0, bonded=False)
    add("globule269", glob.positions.astype(np.float32), glob.types, full, 0)
    add("coil269_w16", sysm.positions.astype(np.float32), sysm.types, full, 0, quant=True)
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 1.6, size=(24, 3)).astype(np.float32)
    add("small_w16", pos, rng.integers(0, 6, size=24), SMALL, 3, quant=True)
    np.savez_compressed(OUT / "flash.npz", **out)


def md_fixture():
    out = {}
    # noise streams, md.py:127-131 / :167-168
    for (seed, rep, step, n) in [(0, 0, 0, 269), (0, 63, 999, 269), (9, 3, 17, 50),
                                 (2 ** 40, 7, 123456789, 269)]:
        g = RMD.make_step_rng(seed, rep, step)
        out[f"noise/{seed}_{rep}_{step}_{n}"] = g.standard_normal((n, 3))
    big = RMD.make_step_rng(5, 1, 2).standard_normal((20000, 3))
    out["noise_big/sha_f32"] = sha(big.astype(np.float32))
    # one BAOA step + half-kick given forces (fp32), md.py:134-172
    rng = np.random.default_rng(4)
    R, N = 3, 40
    pos = rng.uniform(0, 3, size=(R, N, 3)).astype(np.float32)
    vel = rng.normal(0, 0.5, size=(R, N, 3)).astype(np.float32)
    F = rng.normal(0, 300, size=(R, N, 3)).astype(np.float32)
    F2 = rng.normal(0, 300, size=(R, N, 3)).astype(np.float32)
    masses = rng.uniform(50, 150, size=N)
    cfg = RMD.SimConfig(dt_fs=4.0, temperature=300.0, friction=1.0, seed=7)
    st = RMD.SimState(positions=pos, velocities=vel, masses=masses, step=11)
    rngs = [RMD.make_step_rng(7, r, 11) for r in range(R)]
    s1 = RMD.langevin_step(st, F, cfg, rngs)
    s2 = RMD.half_kick(s1, F2, cfg)
    out.update({"step/pos": pos, "step/vel": vel, "step/F": F, "step/F2": F2,
                "step/masses": masses, "step/pos1": s1.positions, "step/vel1": s1.velocities,
                "step/vel2": s2.velocities})
    # prior on a perturbed chain
    chain = RS.generate_system("coil", 30, 2)
    p32 = (chain.positions + rng.normal(0, 0.05, size=chain.positions.shape)).astype(np.float32)
    e, f = RMD.prior_energy_forces(p32, chain.prior)
    out.update({"prior/pos": p32, "prior/energy": e, "prior/forces": f})
    # short trajectories through run_simulation
    import tempfile
    for name, kind, n, sseed, cfgd, pseed, R, steps, stride in [
            ("traj_tiny", "coil", 20, 3, TINY, 2, 3, 20, 1),
            ("traj_tiny_stride3", "coil", 20, 3, TINY, 2, 2, 20, 3),
            ("traj_coil269", "coil", 269, 0, {}, 0, 2, 10, 1)]:
        params = RM.init_params(RM.ModelConfig(**cfgd), pseed)
        sysm = RS.generate_system(kind, n, sseed)
        sim = RMD.SimConfig(dt_fs=4.0, temperature=300.0, friction=1.0, n_steps=steps,
                            n_replicas=R, seed=9, output_stride=5, neighbor_stride=stride)
        with tempfile.TemporaryDirectory() as td:
            res = RMD.run_simulation(params, sysm, sim, td)
            scal = (Path(td) / "scalars.csv").read_text()
            traj = (Path(td) / "trajectory.xyz").read_text()
        out.update({f"{name}/pos": res.final_state.positions,
                    f"{name}/vel": res.final_state.velocities,
                    f"{name}/mean_edges": res.mean_edges, f"{name}/scalars": scal,
                    f"{name}/traj_sha": hashlib.sha256(traj.encode()).hexdigest(),
                    f"{name}/cfg": json.dumps(cfgd), f"{name}/stride": stride,
                    f"{name}/meta": np.array([n, sseed, pseed, R, steps])})
    np.savez_compressed(OUT / "md.npz", **out)


def md_long_fixture():
    """SURVEY §8(c) trajectory bar: 100 fp32 steps of coil-269 (R=2) through
    the reference run_simulation, plus a 16-bit run (quantize_model weights,
    20 steps) for the C3 configuration.  Written to md_long.npz so the
    shorter md.npz fixtures stay byte-stable."""
    import tempfile
    out = {}
    for name, quant, R, steps in [("traj_coil269_100", False, 2, 100),
                                  ("traj_coil269_w16", True, 2, 20)]:
        params = RM.init_params(RM.ModelConfig(), 0)
        if quant:
            params = RQ.quantize_model(params, seed=0)
        sysm = RS.generate_system("coil", 269, 0)
        sim = RMD.SimConfig(dt_fs=4.0, temperature=300.0, friction=1.0, n_steps=steps,
                            n_replicas=R, seed=9, output_stride=10, neighbor_stride=1)
        with tempfile.TemporaryDirectory() as td:
            res = RMD.run_simulation(params, sysm, sim, td)
            scal = (Path(td) / "scalars.csv").read_text()
        # wall_ms (the last column) is measured time; drop it so the fixture
        # is byte-stable across regenerations
        scal = "\n".join(",".join(ln.split(",")[:5]) for ln in scal.splitlines()) + "\n"
        out.update({f"{name}/pos": res.final_state.positions,
                    f"{name}/vel": res.final_state.velocities,
                    f"{name}/mean_edges": res.mean_edges, f"{name}/scalars": scal,
                    f"{name}/quant": quant, f"{name}/cfg": json.dumps({}), f"{name}/stride": 1,
                    f"{name}/meta": np.array([269, 0, 0, R, steps])})
    np.savez_compressed(OUT / "md_long.npz", **out)


def hashes_fixture():
    h = {"numpy": np.__version__}
    for kind, n, seed, bonded in [("coil", 269, 0, True), ("coil", 20, 3, True),
                                  ("globule", 269, 0, False), ("globule", 14, 6, True),
                                  ("helix", 6, 0, True), ("coil", 1000, 0, True)]:
        s = RS.generate_system(kind, n, seed, bonded=bonded)
        h[f"system/{kind}_{n}_{seed}_{int(bonded)}"] = {
            "positions": sha(s.positions), "types": sha(s.types), "masses": sha(s.masses),
            "bonds": sha(s.prior.bonds) if s.prior is not None else None}
    for name, cfg, seed in [("default_0", {}, 0), ("small_3", SMALL, 3), ("tiny_2", TINY, 2)]:
        h[f"params/{name}"] = params_hash(RM.init_params(RM.ModelConfig(**cfg), seed))
    q = RQ.quantize_model(RM.init_params(RM.ModelConfig(), 0), seed=0)
    qh = hashlib.sha256()
    for bp in q.blocks:
        for lin in (bp.pre_linear, *bp.filter_mlp.layers, *bp.post_mlp.layers):
            for a in (lin.weight, lin.scale, lin.bias):
                qh.update(sha(a).encode())
    for lin in q.readout.layers:
        for a in (lin.weight, lin.scale, lin.bias):
            qh.update(sha(a).encode())
    h["quant/default_0"] = qh.hexdigest()
    (OUT / "hashes.json").write_text(json.dumps(h, indent=1, sort_keys=True))


if __name__ == "__main__":
    neighbors_fixture()
    flash_fixture()
    md_fixture()
    md_long_fixture()
    hashes_fixture()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
