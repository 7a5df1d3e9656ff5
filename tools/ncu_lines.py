"""Stall samples and executed instructions per CUDA source line of one kernel
in an ncu --set full report (mixed cuda,sass source page).

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [launch_index]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, kernel, top=40, which=0):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kernel}"]
    raw = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    fname, hdr, func, seen = None, None, None, -1
    agg = defaultdict(lambda: [0, 0, ""])
    cur_line = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            if r[1] != func:
                func = r[1]
                seen += 1
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if seen != which or hdr is None:
            continue
        if r[0]:
            cur_line = (fname, int(r[0]), r[1].strip()[:100])
        if len(r) > 7 and r[2]:
            try:
                s = int(r[4] or 0)
                ie = int(r[7] or 0)
            except ValueError:
                continue
            a = agg[cur_line[:2]]
            a[0] += s
            a[1] += ie
            a[2] = cur_line[2]
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"{func}: {tot} samples")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0]:6d} {100 * v[0] / tot:5.1f}% {v[1]:8d}  {k[0]}:{k[1]}  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
