"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py TAG [CONFIG]
reads gpurun_out/launches_TAG.csv (gpu__time_duration launch list) and
gpurun_out/prof_TAG.ncu-rep (--set full captures), writes
profiles/TAG_summary.md and merges per-kernel DRAM bytes into
profiles/ncu_summary.json under CONFIG (bench.py's config_tag, default
the C2 headline "coil269_rc1.5_fp32_R64"; read by bench.py for
roofline.traffic of the same configuration).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
              "us": 1e-6, "ms": 1e-3, "s": 1.0,
              "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def short(name: str) -> str:
    return name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]


def launch_list(tag):
    p = ROOT / "gpurun_out" / f"launches_{tag}.csv"
    if not p.exists():
        return None
    text = p.read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1.0)
        k = short(r["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    return tot, cnt


def full_set(tag):
    reps = sorted((ROOT / "gpurun_out").glob(f"prof_{tag}*.ncu-rep"))
    res = []
    for p in reps:
        res += _full_one(p)
    return res


def _full_one(p):
    out = subprocess.run(["ncu", "-i", str(p), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, key in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * UNIT_SCALE.get(units[i], 1.0) if units[i] in UNIT_SCALE else v
        res.append(d)
    return res


def main(tag, config="coil269_rc1.5_fp32_R64"):
    lines = [f"# ncu summary `{tag}`", ""]
    ll = launch_list(tag)
    if ll:
        tot, cnt = ll
        T = sum(tot.values())
        lines += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
                  "| kernel | launches | total µs | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| {k} | {cnt[k]} | {v * 1e6:.1f} | {v / T:.3f} |")
        lines.append("")
    fs = full_set(tag)
    summary_path = ROOT / "profiles" / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    if fs:
        keys = [k for _, k in METRICS]
        lines += ["## --set full captures", "", "| kernel | " + " | ".join(keys) + " |",
                  "|---|" + "---|" * len(keys)]
        for d in fs:
            vals = []
            for k in keys:
                v = d.get(k)
                if v is None:
                    vals.append("-")
                elif k == "duration":
                    vals.append(f"{v * 1e6:.1f} µs")
                elif k.startswith("dram_r") or k.startswith("dram_w"):
                    vals.append(f"{v / 1e6:.2f} MB")
                else:
                    vals.append(f"{v:.1f}")
            lines.append(f"| {d['kernel']} | " + " | ".join(vals) + " |")
            name = d["kernel"].replace("k_", "", 1)
            # the default edge kernels carry bench.py's profiler class names
            name = {"edge_bwd_fmws": "edge_bwd", "edge_fwd_ws": "edge_fwd"}.get(name, name)
            for suf in ("_tc", "64"):  # bench.py's profiler classes drop the suffix
                if name.endswith(suf):
                    name = name[:-len(suf)]
            if "dram_read" in d:
                summary.setdefault(config, {})[name] = {"dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0),
                                 "duration_s": d.get("duration"), "tag": tag}
    (ROOT / "profiles").mkdir(exist_ok=True)
    (ROOT / "profiles" / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
    summary_path.write_text(json.dumps(summary, indent=1, sort_keys=True))
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:3])
