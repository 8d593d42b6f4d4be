"""DRAM traffic per launch of each kernel in an `ncu --set full` report, for
bench.py's roofline `traffic` field.

usage: python tools/ncu_traffic.py REPORT.ncu-rep CONFIG OUT.json
Merges {CONFIG: {kernel: {"dram_bytes": read+write per launch, "duration_ns",
"launches"}}} into OUT.json (kernel = name without template arguments)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TUNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}


def main(rep, config, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    it = hdr.index("gpu__time_duration.sum")
    acc = defaultdict(lambda: [0.0, 0.0, 0, 0.0, 0.0, 0.0])
    for r in data:
        name = r[ki].replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = name.replace("void ", "").split("(")[0].split("<")[0].strip()
        b = float(r[ir]) * UNIT[units[ir]] + float(r[iw]) * UNIT[units[iw]]
        t = float(r[it]) * TUNIT[units[it]]
        a = acc[name]
        a[0] += b
        a[1] += t
        a[2] += 1
        for k, op in enumerate(("dfma", "dmul", "dadd")):
            key = f"sm__sass_thread_inst_executed_op_{op}_pred_on.sum"
            if key in hdr:
                try:
                    a[3 + k] += float(r[hdr.index(key)].replace(",", ""))
                except ValueError:
                    pass
    res = json.load(open(out)) if os.path.exists(out) else {}
    res[config] = {k: {"dram_bytes": v[0] / v[2], "duration_ns": v[1] / v[2], "launches": v[2],
                       "dfma": v[3] / v[2], "dmul": v[4] / v[2], "dadd": v[5] / v[2],
                       "source": os.path.basename(rep)}
                   for k, v in acc.items()}
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(*sys.argv[1:4])
