"""Physics known-answer tests of the GPU path, ported from the reference's
own suite: finite-difference forces and the no-edge case
(test_flash.py:118-124, :169-182), permutation / rigid-motion invariance,
net force and torque (test_reference.py:129-178), and the integrator's
identity step, NVE energy conservation and momentum conservation
(test_md.py:86-151).

The reference runs these in fp64 (its "64bit" mode); the B200 path is the
reference's fp32 production precision, so the bars are fp32 ones: energies
carry ~1e-7 relative round-off, which a central difference with step h
turns into ~1e-7 |E| / h of force error (bar 2e-3 relative at h = 2e-3 nm),
and a 1 fs fp32 velocity-Verlet run is held to a total-energy drift of
2e-3 of the kinetic energy it exchanges (momentum to 1e-5 of sum m|v|).  The identity step
is bit-exact, as in the reference.
"""

import ctypes as C

import numpy as np
import pytest

import paper_2602_13140_b200 as P
from oracle import flashcg_oracle as O
from paper_2602_13140_b200.modelparams import ModelConfig, init_params

pytestmark = pytest.mark.gpu

SMALL = ModelConfig(hidden_dim=16, rbf_dim=8, num_blocks=2, cutoff=1.0, num_atom_types=6,
                    filter_hidden_dim=16, readout_hidden_dim=8)
MD_CFG = ModelConfig(hidden_dim=16, rbf_dim=8, num_blocks=2, cutoff=1.2, num_atom_types=8,
                     filter_hidden_dim=16, readout_hidden_dim=8)  # generate_system: 8 types


def instance(seed, n=16):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, 0.8 * n ** (1.0 / 3.0), (n, 3)).astype(np.float32)
    types = rng.integers(0, SMALL.num_atom_types, n)
    return pos, types, init_params(SMALL, seed)


def energy(pos, types, params):
    return P.flash_energy_forces(pos, types, params, P.PipelineMode())


def rotation(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q *= np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def test_forces_match_finite_differences_of_energy():
    pos, types, params = instance(5, n=10)
    out = energy(pos, types, params)
    assert out.forces.shape == pos.shape
    h = 2e-3
    fd = np.zeros(pos.shape, np.float64)
    for i in range(pos.shape[0]):
        for k in range(3):
            e, x = [], []
            for sgn in (1.0, -1.0):
                p = pos.copy()
                p[i, k] = np.float32(p[i, k] + sgn * h)
                e.append(energy(p, types, params).energy)
                x.append(float(p[i, k]))
            fd[i, k] = -(e[0] - e[1]) / (x[0] - x[1])  # the fp32 step actually taken
    # fp32 energy round-off ~1e-7 |E| / h of absolute force noise, plus O(h^2)
    assert O.force_rel_err(out.forces, fd) <= 2e-3


def test_no_edges_energy_matches_oracle_and_forces_vanish():
    pos, types, params = instance(1, n=5)
    spread = pos + (np.arange(5)[:, None] * 50.0).astype(np.float32)
    out = energy(spread, types, params)
    ref = O.energy_forces(spread, types, params)
    assert out.energy == pytest.approx(float(ref[0]), rel=1e-6, abs=1e-6)
    np.testing.assert_array_equal(out.forces, np.zeros_like(out.forces))


def test_permutation_invariance():
    pos, types, params = instance(6, n=30)
    a = energy(pos, types, params)
    perm = np.random.default_rng(0).permutation(pos.shape[0])
    b = energy(pos[perm], types[perm], params)
    assert abs(b.energy - a.energy) <= 1e-5 * max(abs(a.energy), 1.0)
    assert O.force_rel_err(b.forces, a.forces[perm]) <= 1e-5


def test_rigid_motion_invariance_and_force_covariance():
    pos, types, params = instance(7, n=12)
    a = energy(pos, types, params)
    scale = max(abs(a.energy), 1.0)
    rng = np.random.default_rng(7)
    for _ in range(20):
        q = rotation(rng)
        moved = (pos.astype(np.float64) @ q.T + rng.standard_normal(3)).astype(np.float32)
        b = energy(moved, types, params)
        assert abs(b.energy - a.energy) <= 1e-5 * scale
        assert O.force_rel_err(b.forces, a.forces.astype(np.float64) @ q.T) <= 1e-4


def test_net_force_and_torque_vanish():
    pos, types, params = instance(9, n=30)
    f = energy(pos, types, params).forces.astype(np.float64)
    scale = np.max(np.linalg.norm(f, axis=1)) + 1e-30
    assert np.max(np.abs(f.sum(axis=0))) / scale < 1e-4
    c = pos.astype(np.float64) - pos.astype(np.float64).mean(axis=0)
    assert np.max(np.abs(np.cross(c, f).sum(axis=0))) / scale < 1e-4


def test_langevin_identity_when_everything_off():
    # test_md.py:86-95: no force, no friction, no temperature -> identity
    import torch
    from paper_2602_13140_b200 import _lib
    from paper_2602_13140_b200.engine import md_params
    lib = _lib.load()
    p = md_params(1.0, 0.0, 0.0, 0)
    R, N = 1, 2
    pos = torch.ones(R, N, 3, device="cuda")
    vel = torch.zeros(R, N, 3, device="cuda")
    F = torch.zeros_like(pos)
    mass = torch.ones(N, device="cuda")
    noise = torch.empty_like(pos)
    st = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    v = _lib.vp
    _lib.check(lib.fcg_normal_noise(0, 0, v(st), R, N, v(noise), s), "noise")
    _lib.check(lib.fcg_langevin_baoa(C.byref(p), v(mass), R, N, v(F), v(noise), v(pos), v(vel),
                                     s), "baoa")
    assert torch.equal(pos, torch.ones_like(pos)) and torch.equal(vel, torch.zeros_like(vel))


def _nve_engine(R=2, n=12):
    from paper_2602_13140_b200.engine import MDEngine
    from paper_2602_13140_b200.inputs import generate_system
    sysm = generate_system("coil", n, 3)
    params = init_params(MD_CFG, 1)
    eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R, dt_fs=1.0, temperature=0.0,
                   friction=0.0, seed=2)
    rng = np.random.default_rng(4)
    pos = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
    pos += (0.02 * rng.standard_normal(pos.shape)).astype(np.float32)  # off equilibrium
    eng.load_state(pos, np.zeros_like(pos), 0)
    eng.evaluate()
    return eng, np.asarray(sysm.masses, np.float64)


def test_nve_energy_conservation_without_thermostat():
    # test_md.py:98-114 (there: a stretched bond, fp64, 10k steps, 1e-4)
    eng, m = _nve_engine()
    etot, ke_max = [], 0.0
    for _ in range(400):
        eng.run(1)
        vel = eng.vel.double().cpu().numpy()
        ke = 0.5 * np.sum(m[None, :, None] * vel ** 2, axis=(1, 2))
        u = eng.potential.double().cpu().numpy() + eng.prior_e.double().cpu().numpy()
        etot.append(ke + u)
        ke_max = max(ke_max, float(ke.max()))
    etot = np.asarray(etot)
    assert ke_max > 1.0  # the run exchanges energy
    drift = np.max(np.abs(etot - etot[0]), axis=0)
    assert np.all(drift <= 2e-3 * ke_max), (drift, ke_max)


def test_momentum_conserved_without_friction():
    # test_md.py:136-151: sum m v stays at its initial zero
    eng, m = _nve_engine()
    eng.run(200)
    vel = eng.vel.double().cpu().numpy()
    mom = np.sum(m[None, :, None] * vel, axis=1)          # per replica
    scale = np.sum(m[None, :, None] * np.abs(vel), axis=1) + 1e-30
    assert np.max(np.abs(mom) / scale) <= 1e-5
