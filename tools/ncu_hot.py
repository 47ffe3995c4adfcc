"""Hot-spot view of an ncu report: stall reasons, and stall samples
aggregated by CUDA source line (needs -lineinfo + --import-source).

    python tools/ncu_hot.py gpurun_out/prof_X.ncu-rep [N]
"""

import csv
import io
import subprocess
import sys


def main(rep, n=30):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, r = rows[0], rows[2]
    st = []
    for i, k in enumerate(h):
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), k.split("stalled_")[-1]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("stall reasons:", ", ".join(f"{k} {v / tot:.1%}" for v, k in sorted(st, reverse=True)[:8]))
    for key in ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if key in h:
            print(f"  {key} = {r[h.index(key)]} {rows[1][h.index(key)]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    res = []
    fname = "?"
    hdr = None
    for row in csv.reader(io.StringIO(src)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            wi = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or row[0] == "" or len(row) <= wi:
            continue
        try:
            res.append((float(row[wi]), fname, row[0], row[1]))
        except ValueError:
            pass
    T = sum(v for v, *_ in res) or 1
    for v, f, line, text in sorted(res, reverse=True)[:n]:
        print(f"{v / T:6.1%}  {f}:{line:<5} {text.strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
