"""Per-CUDA-source-line executed instructions and stall samples of an ncu
report (needs -lineinfo + --import-source):

    python tools/ncu_lines.py gpurun_out/prof_X.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, n=40):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, res = "?", None, []
    for row in csv.reader(io.StringIO(src)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            ie = hdr.index("Instructions Executed")
            ws = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or not row[0] or len(row) <= max(ie, ws):
            continue
        try:
            res.append((float(row[ie] or 0), float(row[ws] or 0), fname, row[0], row[1]))
        except ValueError:
            pass
    ti = sum(r[0] for r in res) or 1
    ts = sum(r[1] for r in res) or 1
    print(f"total instructions executed {ti:.4g}")
    for i, s, f, line, text in sorted(res, reverse=True)[:n]:
        print(f"{i / ti:6.1%} inst {s / ts:6.1%} stall  {f}:{line:<5} {text.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
