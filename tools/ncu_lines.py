"""Per-source-line instruction counts and stall samples of one kernel in an
ncu report (the cuda,sass correlated source page).

usage: python tools/ncu_lines.py REPORT.ncu-rep [FILE_SUBSTRING] [TOP]
Prints lines sorted by warp instructions executed, with their share and the
warp-stall samples."""
import csv
import io
import subprocess
import sys


def main(rep, fsub="", top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    cur = None
    rows = []
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or cur is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            inst = float(r[hdr.index("Instructions Executed")])
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        rows.append((cur, int(r[0]), r[1], inst, samp))
    tot_i = sum(x[3] for x in rows) or 1.0
    tot_s = sum(x[4] for x in rows) or 1.0
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    for f, ln, src, inst, samp in sorted((x for x in rows if fsub in x[0]), key=lambda x: -x[3])[:top]:
        print(f"{f.split('/')[-1]}:{ln:<5d} inst {inst:11.4g} ({100 * inst / tot_i:5.1f}%)  "
              f"stall {100 * samp / tot_s:5.1f}%  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "",
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)
