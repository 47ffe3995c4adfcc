"""Top SASS instructions of an ncu report for one stall reason, with the
instructions just before each (to see which load a scoreboard wait is on).

    python tools/sass_stalls.py gpurun_out/prof_X.ncu-rep [reason=long_sb] [N=12] [ctx=4]
"""
import csv
import io
import subprocess
import sys


def main(rep, reason="long_sb", n=12, ctx=4):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = rows[2:]
    ia, isrc, col = h.index("Address"), h.index("Source"), h.index("stall_" + reason)

    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0

    tot = sum(f(r[col]) for r in data) or 1.0
    for i in sorted(range(len(data)), key=lambda i: -f(data[i][col]))[:n]:
        print(f"{100 * f(data[i][col]) / tot:5.1f}%  {data[i][ia]}  {data[i][isrc][:90]}")
        for j in range(max(0, i - ctx), i):
            print(f"          {data[j][ia]}  {data[j][isrc][:90]}")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 else "long_sb", int(a[2]) if len(a) > 2 else 12,
         int(a[3]) if len(a) > 3 else 4)
