"""Aggregate an ncu report's per-SASS stall samples by CUDA source line.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep paper_2412_10287_b200/librpq_b200.so [kernel]

COL=<source-page column> replaces "Instructions Executed" as the second
figure (e.g. COL="L2 Theoretical Sectors Global"); SORT=col orders by it.
ncu's source page of a -lineinfo build lists SASS with stall samples; the
cubin inside the .so carries the line table (nvdisasm --print-line-info), so
function offsets map to lines of csrc/*.cuh.
"""

import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def line_map(so, kernel_substr):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, check=True, capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cubin)],
                         capture_output=True, text=True).stdout
    out, infn, cur = {}, False, None
    for ln in dis.splitlines():
        if ln.startswith("\t.section\t.text.") or ln.startswith(".text."):
            infn = kernel_substr in ln
        if not infn:
            continue
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if "//## File" in ln and m:
            cur = (m.group(1), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]+)\*/", ln)
        if m and cur is not None:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    rep, so = sys.argv[1], os.path.abspath(sys.argv[2])
    kernel = sys.argv[3] if len(sys.argv) > 3 else "ssr_kernel"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    ii = h.index(os.environ.get("COL", "Instructions Executed"))
    addrs = [(int(r[0], 16), int(r[si] or 0), int(float(r[ii] or 0))) for r in rows[2:] if r and r[0].startswith("0x")]
    base = min(a for a, _, _ in addrs)
    lm = line_map(so, kernel)
    src_path = None
    by_line = defaultdict(lambda: [0, 0])
    for a, smp, ins in addrs:
        ln = lm.get(a - base)
        by_line[ln][0] += smp
        by_line[ln][1] += ins
    tot = sum(v[0] for v in by_line.values())
    srcs = {}

    def text_of(key):
        if not key:
            return "?", "?"
        path, ln = key
        if path not in srcs:
            cand = path if os.path.exists(path) else os.path.join(os.path.dirname(so), "csrc", os.path.basename(path))
            srcs[path] = open(cand).read().splitlines() if os.path.exists(cand) else []
        lines = srcs[path]
        return f"{os.path.basename(path)}:{ln}", (lines[ln - 1].strip()[:80] if ln <= len(lines) else "?")

    print(f"total samples {tot}")
    col = 1 if os.environ.get("SORT") == "col" else 0
    for key, (smp, ins) in sorted(by_line.items(), key=lambda kv: -kv[1][col])[:int(os.environ.get("TOP", 30))]:
        loc, text = text_of(key)
        print(f"{smp:7d} {100.0 * smp / max(tot, 1):5.1f}% {ins:10d}  {loc}: {text}")


if __name__ == "__main__":
    main()
