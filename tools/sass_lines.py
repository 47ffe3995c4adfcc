"""Static SASS instruction count per CUDA source line of one kernel.

    python tools/sass_lines.py build/fcg/edge_tc.o KERNEL_SUBSTRING [N]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile


def main(obj, kern, n=40):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d,
                       capture_output=True)
        cubins = [f for f in os.listdir(d) if f.endswith(".cubin")]
        out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubins[0])],
                             capture_output=True, text=True).stdout
    cur, fn, cnt = None, None, collections.Counter()
    for line in out.splitlines():
        m = re.search(r"\.text\.(\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        if fn and kern in fn and re.match(r"\s+/\*[0-9a-f]{4}\*/", line) and cur:
            cnt[cur] += 1
    print("total", sum(cnt.values()))
    for (f, l), c in sorted(cnt.items(), key=lambda x: -x[1])[:n]:
        print(c, f, l)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
