"""Executed local-memory instructions (register spills: LDL/STL) of a kernel
in an ncu report, by CUDA source line.

    python tools/ncu_spills.py gpurun_out/prof.ncu-rep paper_2412_10287_b200/librpq_b200.so [kernel]
"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import line_map  # noqa: E402


def main():
    rep, so = sys.argv[1], os.path.abspath(sys.argv[2])
    kernel = sys.argv[3] if len(sys.argv) > 3 else "ssr_kernel"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    si, ii = h.index("Source"), h.index("Instructions Executed")
    recs = [(int(r[0], 16), r[si], int(float(r[ii] or 0))) for r in rows[2:] if r and r[0].startswith("0x")]
    base = min(a for a, _, _ in recs)
    lm = line_map(so, kernel)
    by = defaultdict(lambda: [0, 0])
    for a, src, n in recs:
        op = src.split()[0] if src.split() else ""
        if op.startswith("@"):
            op = src.split()[1]
        if op.startswith("LDL") or op.startswith("STL"):
            key = lm.get(a - base)
            by[key][0 if op.startswith("LDL") else 1] += n
    tot = [sum(v[0] for v in by.values()), sum(v[1] for v in by.values())]
    print(f"executed LDL {tot[0]}  STL {tot[1]}")
    for key, (l, s_) in sorted(by.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:25]:
        print(f"{l:10d} {s_:10d}  {key}")


if __name__ == "__main__":
    main()
