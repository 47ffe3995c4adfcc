"""Top CUDA source lines per stall reason of an ncu report.

    python tools/ncu_stalls.py gpurun_out/prof_X.ncu-rep [reasons...]
"""
import csv
import io
import subprocess
import sys


def main(rep, reasons):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    hdr, res, fname = None, [], "?"
    for row in csv.reader(io.StringIO(src)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0]:
            continue
        d = dict(zip(hdr, row))
        res.append((d, fname, row[0], row[1][:80]))
    for r in reasons:
        key = "stall_" + r
        tot = sum(float(d.get(key) or 0) for d, *_ in res) or 1
        print("==", r)
        for d, f, line, text in sorted(res, key=lambda x: -float(x[0].get(key) or 0))[:8]:
            print(f"{float(d.get(key) or 0) / tot:6.1%} {f}:{line} {text}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:] or ["long_sb", "no_inst", "wait"])
