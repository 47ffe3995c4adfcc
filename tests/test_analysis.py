"""Trajectory analysis: the oracle pinned against the
reference's own outputs (tests/golden/make_analysis_golden.py), the host
side of paper_2602_13140_b200.analysis on CPU, and the CUDA kernels
(fcg_kabsch / fcg_native_q / fcg_gdt_counts) against both on the GPU.

Bars: GDT-TS best counts, contact sets, edge counts and degrees exact;
rotations/translations <= 1e-10, RMSD <= 1e-12 and Q <= 1e-12 (fp64, a
different but exact superposition algorithm and reduction order);
savitzky_golay <= 1e-10 (the reference test's bar against scipy).
"""

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import analysis_oracle as AO
import paper_2602_13140_b200.analysis as A

GOLD = np.load(Path(__file__).parent / "golden" / "analysis.npz")
CASES = ("c64", "c269")


# ---- oracle pinned to the reference (CPU) ----------------------------------------

@pytest.mark.parametrize("tag", CASES)
def test_oracle_matches_reference_metrics(tag):
    native, frames = GOLD[f"{tag}_native"], GOLD[f"{tag}_frames"]
    pairs, r0 = AO.contacts(native)
    np.testing.assert_array_equal(pairs, GOLD[f"{tag}_pairs"])
    np.testing.assert_array_equal(r0, GOLD[f"{tag}_ref_dist"])
    for k, f in enumerate(frames):
        rot, tr, r = AO.kabsch(f, native)
        np.testing.assert_array_equal(rot, GOLD[f"{tag}_rot"][k])
        np.testing.assert_array_equal(tr, GOLD[f"{tag}_trans"][k])
        assert r == GOLD[f"{tag}_rmsd"][k]
        assert AO.native_q(f, pairs, r0) == GOLD[f"{tag}_q"][k]
        assert AO.gdt_ts(f, native) == GOLD[f"{tag}_gdt"][k]
    gs = AO.graph_stats(frames, 1.5)
    for key, v in gs.items():
        np.testing.assert_array_equal(v, GOLD[f"{tag}_graph_{key}"])


def test_oracle_series_and_degenerate_cases():
    np.testing.assert_array_equal(AO.savgol(GOLD["savgol_in"], 11, 3), GOLD["savgol_out"])
    assert AO.largest_metastable_q(GOLD["lmq_bimodal"]) == float(GOLD["lmq_bimodal_value"])
    assert AO.gdt_ts(GOLD["gdt_disp_x"], GOLD["gdt_disp_ref"]) == float(GOLD["gdt_disp_value"])
    line = np.zeros((6, 3))
    line[:, 0] = np.arange(6)
    with pytest.raises(AO.Degenerate):
        AO.kabsch(line, line)


# ---- host side of the product module (CPU) ---------------------------------------

def test_build_contacts_and_windows_match_reference():
    for tag in CASES:
        cs = A.build_contacts(GOLD[f"{tag}_native"])
        np.testing.assert_array_equal(cs.pairs, GOLD[f"{tag}_pairs"])
        np.testing.assert_array_equal(cs.ref_dist, GOLD[f"{tag}_ref_dist"])
        assert cs.count == GOLD[f"{tag}_pairs"].shape[0]
    w = A.gdt_windows(269)
    assert w.shape == (1 + (269 - 134 + 1) + (269 - 67 + 1), 2)
    assert tuple(w[0]) == (0, 269) and tuple(w[1]) == (0, 134) and tuple(w[-1]) == (202, 67)
    assert A.gdt_windows(5).tolist() == [[0, 5], [0, 3], [1, 3], [2, 3]]


def test_series_analysis_matches_reference():
    np.testing.assert_allclose(A.savitzky_golay(GOLD["savgol_in"], 11, 3), GOLD["savgol_out"],
                               rtol=0, atol=1e-10)
    assert A.largest_metastable_q(GOLD["lmq_bimodal"]) == float(GOLD["lmq_bimodal_value"])
    assert A.largest_metastable_q(np.full(100, 0.9)) == 0.9
    x = np.arange(40, dtype=float)
    for coeffs in ([1.0], [0.5, -2.0], [0.1, 0.3, -0.02], [0.01, -0.1, 0.05, 0.002]):
        y = np.polyval(coeffs, x)
        np.testing.assert_allclose(A.savitzky_golay(y, 11, 3), y, atol=1e-8)
    with pytest.raises(ValueError):
        A.savitzky_golay(np.zeros(30), window=10, order=3)
    with pytest.raises(ValueError):
        A.savitzky_golay(np.zeros(30), window=3, order=3)
    with pytest.raises(ValueError):
        A.largest_metastable_q(np.zeros(0))


def test_metrics_csv_and_trajectory_io_match_reference(tmp_path):
    series = A.MetricSeries(steps=np.array([0, 10, 20]), rmsd=np.array([0.0, 0.123456789, 1.5]),
                            q=np.array([1.0, 0.87654321, 0.25]), edges=np.array([100, 98, 97]),
                            gdt=np.array([1.0, 0.75, 0.125]))
    A.write_metrics_csv(series, tmp_path / "m.csv")
    assert (tmp_path / "m.csv").read_bytes() == GOLD["metrics_csv"].tobytes()
    (tmp_path / "t.xyz").write_bytes(GOLD["traj_text"].tobytes())
    fr = A.read_trajectory(tmp_path / "t.xyz")
    assert [f[0] for f in fr] == GOLD["traj_steps"].tolist()
    assert [f[1] for f in fr] == GOLD["traj_replicas"].tolist()
    np.testing.assert_array_equal(np.asarray([f[2] for f in fr]), GOLD["traj_types"])
    np.testing.assert_array_equal(np.asarray([f[3] for f in fr]), GOLD["traj_pos"])
    (tmp_path / "e.xyz").write_text("\n\n")
    with pytest.raises(ValueError):
        A.read_trajectory(tmp_path / "e.xyz")
    with pytest.raises(ValueError):
        A.MetricSeries(steps=np.arange(3), rmsd=np.zeros(2), q=np.zeros(3), edges=np.zeros(3))


# ---- CUDA kernels (GPU) -------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("tag", CASES)
def test_gpu_kabsch_q_gdt_match_reference(tag):
    native, frames = GOLD[f"{tag}_native"], GOLD[f"{tag}_frames"]
    rot, tr, rms, deg = A.kabsch_batch(frames, native)
    assert not deg.any()
    np.testing.assert_allclose(rot, GOLD[f"{tag}_rot"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(tr, GOLD[f"{tag}_trans"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(rms, GOLD[f"{tag}_rmsd"], rtol=1e-12, atol=1e-12)
    cs = A.ContactSet(GOLD[f"{tag}_pairs"], GOLD[f"{tag}_ref_dist"])
    np.testing.assert_allclose(A.fraction_native_contacts_batch(frames, cs), GOLD[f"{tag}_q"],
                               rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(A.gdt_ts_batch(frames, native), GOLD[f"{tag}_gdt"])
    gs = A.graph_stats(frames, 1.5)
    for key in ("edges", "max_degree", "max_span"):
        np.testing.assert_array_equal(gs[key], GOLD[f"{tag}_graph_{key}"])
    for key in ("mean_degree", "mean_span"):
        np.testing.assert_allclose(gs[key], GOLD[f"{tag}_graph_{key}"], rtol=1e-12)
    m = A.compute_metrics([(10 * k, 0, None, f) for k, f in enumerate(frames)], native, 1.5,
                          with_gdt=True)
    np.testing.assert_array_equal(m.steps, 10 * np.arange(len(frames)))
    np.testing.assert_allclose(m.rmsd, GOLD[f"{tag}_rmsd"], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(m.gdt, GOLD[f"{tag}_gdt"])
    np.testing.assert_array_equal(m.edges, GOLD[f"{tag}_graph_edges"])


@pytest.mark.gpu
def test_gpu_kabsch_known_answers():
    # test_analysis.py:34-95 of the reference
    rng = np.random.default_rng(1)
    for _ in range(10):
        x = rng.standard_normal((15, 3))
        q, r = np.linalg.qr(rng.standard_normal((3, 3)))
        q *= np.sign(np.diag(r))
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        t = rng.standard_normal(3)
        rot, trans, rr = A.kabsch_align(x, x @ q.T + t)
        assert rr <= 1e-10
        np.testing.assert_allclose(rot, q, atol=1e-9)
        np.testing.assert_allclose(trans, t, atol=1e-9)
    x = rng.standard_normal((12, 3))
    rot, trans, rr = A.kabsch_align(x, x)
    np.testing.assert_allclose(rot, np.eye(3), atol=1e-12)
    assert rr <= 1e-12
    y = x.copy()
    y[:, 2] = -y[:, 2]  # mirror image: still a proper rotation
    rot, _, _ = A.kabsch_align(x, y)
    assert np.linalg.det(rot) == pytest.approx(1.0, abs=1e-10)
    with pytest.raises(A.DegenerateStructureError):
        A.kabsch_align(np.zeros((2, 3)), np.zeros((2, 3)))
    line = np.zeros((6, 3))
    line[:, 0] = np.arange(6)
    with pytest.raises(A.DegenerateStructureError):
        A.kabsch_align(line, line)
    with pytest.raises(A.DegenerateStructureError):
        A.rmsd_batch(np.stack([x[:6], line]), line)
    with pytest.raises(ValueError):
        A.kabsch_align(np.zeros((5, 3)), np.zeros((6, 3)))


@pytest.mark.gpu
def test_gpu_q_and_gdt_known_answers():
    cs = A.ContactSet(pairs=np.array([[0, 1]]), ref_dist=np.array([0.5]))
    q = A.fraction_native_contacts(np.array([[0.0, 0, 0], [0.5, 0, 0]]), cs)
    assert q == pytest.approx(1.0 / (1.0 + math.exp(-2.5)), abs=1e-12)
    assert A.fraction_native_contacts(np.array([[0.0, 0, 0], [50.0, 0, 0]]), cs) == \
        pytest.approx(0.0, abs=1e-12)
    assert A.fraction_native_contacts(np.array([[0.0, 0, 0], [0.75, 0, 0]]), cs) == \
        pytest.approx(0.5, abs=1e-12)
    with pytest.raises(ValueError):
        A.fraction_native_contacts(np.zeros((4, 3)), A.ContactSet(np.zeros((0, 2), np.int64),
                                                                  np.zeros(0)))
    x = np.random.default_rng(0).standard_normal((20, 3))
    assert A.gdt_ts(x, x) == 1.0
    assert A.gdt_ts(GOLD["gdt_disp_x"], GOLD["gdt_disp_ref"]) == float(GOLD["gdt_disp_value"])
    with pytest.raises(A.DegenerateStructureError):
        A.gdt_ts(np.zeros((2, 3)), np.zeros((2, 3)))
