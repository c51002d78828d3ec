#!/usr/bin/env python3
"""Per-CUDA-source-line warp-stall samples (and shared-memory excess
wavefronts) of an ncu report, from the cuda,sass source view: top N lines.

    python profiles/ncu_lines.py <report.ncu-rep> [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    per, total, fname, hdr = {}, 0, "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 2:
            continue
        if r[0]:  # CUDA source line row (aggregated over its SASS)
            try:
                s = int(float(r[4] or 0))
            except ValueError:
                continue
            try:
                ex = int(float(r[hdr.index("L1 Wavefronts Shared Excessive")] or 0))
            except (ValueError, IndexError):
                ex = 0
            total += s
            key = (fname, r[0], r[1].strip()[:80])
            a = per.setdefault(key, [0, 0])
            a[0] += s
            a[1] += ex
    print(f"# {rep}: {total} stall samples")
    for (f, line, txt), (s, ex) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100.0 * s / max(total, 1):6.2f}%  {f}:{line:<5} smem-excess {ex:>10}  {txt}")


if __name__ == "__main__":
    main()
