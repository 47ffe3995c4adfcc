"""Pin the CPU oracle against golden vectors produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import json

import numpy as np
import pytest

from helpers import params_for
from oracle import flashcg_oracle as O
from paper_2602_13140_b200.inputs import generate_system
from paper_2602_13140_b200.modelparams import ModelConfig, init_params


def test_neighbor_cases_bit_exact(golden):
    g = golden["neighbors"]
    names = g.cases("src")
    assert len(names) >= 30
    for name in names:
        c = g.case(name)
        src, dst = O.neighbor_list(c["pos"], float(c["rc"]))
        np.testing.assert_array_equal(src, c["src"], err_msg=name)
        np.testing.assert_array_equal(dst, c["dst"], err_msg=name)
        n = c["pos"].shape[0]
        for key, ptrk, permk in ((dst, "dptr", "dperm"), (src, "sptr", "sperm")):
            ptr, perm = O.group(key, n)
            np.testing.assert_array_equal(ptr, c[ptrk], err_msg=name)
            np.testing.assert_array_equal(perm, c[permk], err_msg=name)


def test_neighbor_adversarial_association(golden):
    g = golden["neighbors"]
    pairs, rc, edge = g["adversarial/pairs"], float(g["adversarial/rc"]), g["adversarial/edge"]
    got = np.array([O.neighbor_list(p, rc)[0].size > 0 for p in pairs])
    np.testing.assert_array_equal(got, edge)
    # the alternative association would disagree on a large share of them
    alt = []
    for p in pairs:
        dx, dy, dz = p[0] - p[1]
        alt.append((dx * dx + dy * dy) + dz * dz < rc * rc)
    assert np.mean(np.array(alt) != edge) > 0.2


def test_known_answer_edge_counts(golden):
    g = golden["neighbors"]
    expect = {"two_beads": 2, "cutoff_strict": 0, "single": 0, "spread_line": 0,
              "triangle": 6, "coincident": 12}
    for name, e in expect.items():
        assert g[f"{name}/src"].size == e


def test_group_hand_examples():
    ptr, perm = O.group(np.array([1, 1, 0]), 2)
    np.testing.assert_array_equal(ptr, [0, 1, 3])
    np.testing.assert_array_equal(perm, [2, 0, 1])
    ptr, perm = O.group(np.array([0, 1, 2]), 3)
    np.testing.assert_array_equal(ptr, [0, 1, 2, 3])
    np.testing.assert_array_equal(perm, [0, 1, 2])


def test_segment_sum_hand_examples():
    v = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    np.testing.assert_array_equal(O.segment_sum(v, np.array([0, 2, 3])), [[4, 6], [5, 6]])
    np.testing.assert_array_equal(O.segment_sum(np.array([[1.0], [2.0]]), np.array([0, 0, 2, 2])),
                                  [[0], [3], [0]])
    out = O.segment_sum(np.zeros((0, 3)), np.array([0, 0, 0]))
    assert out.shape == (2, 3) and np.all(out == 0)


@pytest.mark.parametrize("name", ["small0", "small1", "small2", "small3", "small64", "star",
                                  "no_edges", "coil269", "globule269", "small_w16",
                                  "coil269_w16"])
def test_flash_energy_forces(golden, name):
    c = golden["flash"].case(name)
    params = params_for(c)
    e, pa, f = O.energy_forces(c["pos"], c["types"], params)
    tol = 1e-12 if c["pos"].dtype == np.float64 else 2e-6
    assert O.energy_rel_err(e, float(c["energy"]), c["per_atom"]) <= tol
    assert O.force_rel_err(f, c["forces"]) <= tol
    # and the oracle sits within the reference's own flash-vs-reference spread
    assert O.force_rel_err(f, c["ref_forces"]) <= (1e-9 if tol < 1e-9 else 2e-4)


def test_noise_streams_bit_exact(golden):
    g = golden["md"]
    keys = [k for k in g._z.files if k.startswith("noise/")]
    assert len(keys) == 4
    for k in keys:
        seed, rep, step, n = (int(x) for x in k.split("/")[1].split("_"))
        np.testing.assert_array_equal(O.noise(seed, rep, step, n, dtype=np.float64), g[k])


def test_one_step_bit_exact(golden):
    g = golden["md"]
    R = g["step/pos"].shape[0]
    N = g["step/pos"].shape[1]
    xi = np.stack([O.noise(7, r, 11, N) for r in range(R)])
    r1, v1 = O.baoa(g["step/pos"], g["step/vel"], g["step/F"], g["step/masses"], xi, 4.0, 300.0,
                    1.0)
    np.testing.assert_array_equal(r1, g["step/pos1"])
    np.testing.assert_array_equal(v1, g["step/vel1"])
    v2 = O.half_kick(v1, g["step/F2"], g["step/masses"], 4.0)
    np.testing.assert_array_equal(v2, g["step/vel2"])


def test_prior_bit_exact(golden):
    g = golden["md"]
    chain = generate_system("coil", 30, 2)
    e, f = O.prior_energy_forces(g["prior/pos"], chain.prior)
    assert e == float(g["prior/energy"])
    np.testing.assert_array_equal(f, g["prior/forces"])


@pytest.mark.parametrize("name", ["traj_tiny", "traj_tiny_stride3", "traj_coil269"])
def test_trajectory_matches_reference(golden, name):
    c = golden["md"].case(name)
    n, sseed, pseed, R, steps = (int(x) for x in c["meta"])
    sysm = generate_system("coil", n, sseed)
    params = init_params(ModelConfig(**json.loads(str(c["cfg"]))), pseed)
    pos0 = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
    pos, vel, *_ = O.run_md(params, sysm.types, sysm.masses, sysm.prior, pos0,
                            np.zeros_like(pos0), steps, seed=9,
                            neighbor_stride=int(c["stride"]))
    # the oracle restates the same numpy ops: identical trajectories
    np.testing.assert_array_equal(pos, c["pos"])
    np.testing.assert_array_equal(vel, c["vel"])


@pytest.mark.parametrize("name", ["traj_coil269_100", "traj_coil269_w16"])
def test_long_trajectory_matches_reference(golden, name):
    # SURVEY §8(c) 100-step bar (fp32) and the C3 16-bit run: the oracle
    # must reproduce the reference's run_simulation bit for bit before it
    # is trusted as the GPU's checker on these lengths
    from helpers import quantized
    c = golden["md_long"].case(name)
    n, sseed, pseed, R, steps = (int(x) for x in c["meta"])
    sysm = generate_system("coil", n, sseed)
    params = init_params(ModelConfig(), pseed)
    if bool(c["quant"]):
        params = quantized(params)
    pos0 = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
    pos, vel, *_ = O.run_md(params, sysm.types, sysm.masses, sysm.prior, pos0,
                            np.zeros_like(pos0), steps, seed=9, workers=R)
    np.testing.assert_array_equal(pos, c["pos"])
    np.testing.assert_array_equal(vel, c["vel"])
