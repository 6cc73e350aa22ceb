#!/usr/bin/env python3
"""Per-source-line breakdown of an ncu report (cuda,sass source view).

usage: ncu_lines.py REPORT.ncu-rep [TOP]

Prints, per (file, line) with metrics, warp-stall samples, warp-level
instructions executed, average active threads per instruction, and the
source text; sorted by stall samples.  Needs the report captured with
--import-source on and a -lineinfo build.
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = []
    fname = "?"
    header = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname = os.path.basename(rec[1])
            header = None
            continue
        if rec[0] == "Function Name":
            continue
        if rec[0] == "Line No":
            header = rec
            continue
        if header is None:
            continue
        try:
            line = int(rec[0])
        except ValueError:
            continue
        def col(name):
            i = header.index(name)
            v = rec[i]
            try:
                return float(v)
            except ValueError:
                return 0.0
        samp = col("Warp Stall Sampling (All Samples)")
        extra = {k: col(k) for k in ("stall_wait", "stall_long_sb", "stall_short_sb", "stall_no_inst", "stall_selected")
                 if k in header}
        inst = col("Instructions Executed")
        thr = col("Thread Instructions Executed")
        if samp == 0 and inst == 0:
            continue
        rows.append((samp, inst, thr, fname, line, rec[1].strip()[:60], extra))
    tot_s = sum(r[0] for r in rows) or 1
    tot_i = sum(r[1] for r in rows) or 1
    tot_t = sum(r[2] for r in rows)
    print(f"total samples {tot_s:.0f}  warp inst {tot_i:.3g}  avg threads {tot_t / tot_i:.1f}")
    keys = ("stall_wait", "stall_long_sb", "stall_short_sb", "stall_no_inst", "stall_selected")
    tots = {k: sum(r[6].get(k, 0) for r in rows) for k in keys}
    print("stall totals (% of samples):", {k[6:]: round(100 * v / tot_s, 1) for k, v in tots.items()})
    print(f"{'samp%':>6} {'inst%':>6} {'thr':>5} {'wait':>5} {'lsb':>5} {'ssb':>5} {'noin':>5}  location")
    for s, i, t, f, l, src, ex in sorted(rows, key=lambda r: -r[0])[:top]:
        e = [100 * ex.get(k, 0) / tot_s for k in keys[:4]]
        print(f"{100 * s / tot_s:6.2f} {100 * i / tot_i:6.2f} {t / i if i else 0:5.1f} "
              f"{e[0]:5.2f} {e[1]:5.2f} {e[2]:5.2f} {e[3]:5.2f}  {f}:{l}  {src}")


if __name__ == "__main__":
    main()
