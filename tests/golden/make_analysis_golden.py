"""Golden fixtures for trajectory analysis, produced by
running the REFERENCE (flashcg.analysis) itself.

Run here, where /root/reference exists (it does not on the GPU box):
    python tests/golden/make_analysis_golden.py
Writes tests/golden/analysis.npz (committed).  tests/test_analysis.py pins
oracle/analysis_oracle.py against it on CPU and checks the GPU module
(paper_2602_13140_b200/analysis.py) against it on the GPU.
"""

from __future__ import annotations

import io
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from flashcg import analysis as RA  # noqa: E402
from flashcg import systems as RS  # noqa: E402


def rotation(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q *= np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def frames_for(native, rng, amps):
    out = []
    for a in amps:
        x = native + a * rng.standard_normal(native.shape)
        out.append(x @ rotation(rng).T + rng.standard_normal(3))
    return np.asarray(out)


def main():
    out = {}
    rng = np.random.default_rng(42)
    for tag, n, amps in (("c64", 64, (0.0, 0.02, 0.05, 0.1, 0.2, 0.4, 1.0, 3.0)),
                         ("c269", 269, (0.0, 0.05, 0.3))):
        native = RS.generate_system("coil", n, 0).positions.astype(np.float64)
        frames = frames_for(native, rng, amps)
        contacts = RA.build_contacts(native)
        out[f"{tag}_native"] = native
        out[f"{tag}_frames"] = frames
        out[f"{tag}_pairs"] = contacts.pairs.astype(np.int64)
        out[f"{tag}_ref_dist"] = contacts.ref_dist
        rots, trs, rms = zip(*(RA.kabsch_align(f, native) for f in frames))
        out[f"{tag}_rot"], out[f"{tag}_trans"], out[f"{tag}_rmsd"] = (
            np.asarray(rots), np.asarray(trs), np.asarray(rms))
        out[f"{tag}_q"] = np.array([RA.fraction_native_contacts(f, contacts) for f in frames])
        out[f"{tag}_gdt"] = np.array([RA.gdt_ts(f, native) for f in frames])
        gs = RA.graph_stats(frames, 1.5)
        for k, v in gs.items():
            out[f"{tag}_graph_{k}"] = v
    # GDT single displaced bead (test_analysis.py:177-188)
    r7 = np.random.default_rng(7)
    ref = r7.standard_normal((20, 3))
    x = ref.copy()
    x[5] += np.array([0.3, 0.0, 0.0])
    out["gdt_disp_ref"], out["gdt_disp_x"] = ref, x
    out["gdt_disp_value"] = np.array(RA.gdt_ts(x, ref))
    # series analysis
    r10 = np.random.default_rng(10)
    y = r10.standard_normal(64)
    out["savgol_in"], out["savgol_out"] = y, RA.savitzky_golay(y, 11, 3)
    r11 = np.random.default_rng(11)
    bimodal = np.clip(np.concatenate([r11.normal(0.30, 0.05, 6000),
                                      r11.normal(0.85, 0.04, 3000)]), 0, 1)
    out["lmq_bimodal"], out["lmq_bimodal_value"] = bimodal, np.array(
        RA.largest_metastable_q(bimodal))
    # metrics CSV and trajectory parsing
    series = RA.MetricSeries(steps=np.array([0, 10, 20]), rmsd=np.array([0.0, 0.123456789, 1.5]),
                             q=np.array([1.0, 0.87654321, 0.25]), edges=np.array([100, 98, 97]),
                             gdt=np.array([1.0, 0.75, 0.125]))
    with tempfile.TemporaryDirectory() as d:
        RA.write_metrics_csv(series, Path(d) / "m.csv")
        out["metrics_csv"] = np.frombuffer((Path(d) / "m.csv").read_bytes(), dtype=np.uint8)
        buf = io.StringIO()
        for step, rep, pos in ((0, 0, out["c64_frames"][1]), (10, 3, out["c64_frames"][2])):
            buf.write(f"{pos.shape[0]}\nstep={step} replica={rep}\n")
            for i, p in enumerate(pos):
                buf.write(f"B{i % 8} {p[0]:.9f} {p[1]:.9f} {p[2]:.9f}\n")
        (Path(d) / "t.xyz").write_text(buf.getvalue())
        out["traj_text"] = np.frombuffer(buf.getvalue().encode(), dtype=np.uint8)
        fr = RA.read_trajectory(Path(d) / "t.xyz")
        out["traj_steps"] = np.array([f[0] for f in fr])
        out["traj_replicas"] = np.array([f[1] for f in fr])
        out["traj_types"] = np.asarray([f[2] for f in fr])
        out["traj_pos"] = np.asarray([f[3] for f in fr])
    np.savez_compressed(OUT / "analysis.npz", **out)
    print("wrote", OUT / "analysis.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
