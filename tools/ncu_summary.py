"""Summarise ncu artefacts for profiles/: per-kernel duration, FP64 pipe and
issue utilisation, DRAM bytes, occupancy, top stall reasons (from a
--set full report), and per-kernel share of the step (from a launch list)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads/warp"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
     "tensor pipe IMMA % (active)"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.sum", "IMMA/UTCIMMA warp instr"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread instr"),
    ("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread instr"),
    ("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread instr"),
]
# extra counters the profiling runs add to --set full (tools/refresh_profiles.sh)
EXTRA_METRICS = ",".join(k for k, _ in KEYS[-6:])
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6,
        "GB": 1e9}
TUNIT = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3, "s": 1.0}


def _num(r, hdr, units, key, scale=None):
    if key not in hdr:
        return None
    i = hdr.index(key)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return None
    if scale is not None:
        if units[i] not in scale:
            return None
        v *= scale[units[i]]
    return v


def full_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    lines = []
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        lines.append(f"### {name}")
        for k, lab in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"- {lab}: {r[i]} {units[i]}")
        # derived: achieved FP64 FLOP/s (2 per DFMA) and DRAM GB/s
        t = _num(r, hdr, units, "gpu__time_duration.sum", TUNIT)
        fma_, mul_, add_ = (_num(r, hdr, units, f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum")
                            for o in ("dfma", "dmul", "dadd"))
        if t and fma_ is not None and mul_ is not None and add_ is not None:
            fl = 2.0 * fma_ + mul_ + add_
            lines.append(f"- FP64 flops executed: {fl:.4g} -> {fl / t / 1e12:.3f} TFLOP/s")
        rb = _num(r, hdr, units, "dram__bytes_read.sum", UNIT)
        wb = _num(r, hdr, units, "dram__bytes_write.sum", UNIT)
        if t and rb is not None and wb is not None:
            lines.append(f"- DRAM read+write: {(rb + wb) / t / 1e9:.1f} GB/s")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                nm = h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
                if nm != "selected":
                    st.append((v, nm))
        st.sort(reverse=True)
        lines.append("- top stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]))
        lines.append("")
    return "\n".join(lines)


def launch_list(path, skip_prefix=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    lines = ["| kernel | launches | total ns | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / s:.1f}% |")
    return "\n".join(lines)


def rederive(md_path):
    """Recompute the derived lines (FP64 TFLOP/s, DRAM GB/s) of a summary
    written by full_report from its raw lines (duration, DFMA/DMUL/DADD
    thread instructions, DRAM bytes)."""
    out, cur = [], {}
    for line in open(md_path).read().split("\n"):
        if line.startswith("### "):
            cur = {}
        if line.startswith("- FP64 flops executed") or line.startswith("- DRAM read+write"):
            continue
        out.append(line)
        if not line.startswith("- ") or ":" not in line:
            continue
        lab, val = line[2:].split(":", 1)
        parts = val.split()
        if not parts:
            continue
        try:
            v = float(parts[0])
        except ValueError:
            continue
        u = parts[1] if len(parts) > 1 else ""
        cur[lab] = v * TUNIT.get(u, UNIT.get(u, 1.0)) if lab in ("duration", "dram read", "dram write") else v
        if lab == "DADD thread instr" and "duration" in cur:
            fl = 2.0 * cur.get("DFMA thread instr", 0.0) + cur.get("DMUL thread instr", 0.0) + v
            out.append(f"- FP64 flops executed: {fl:.4g} -> {fl / cur['duration'] / 1e12:.3f} TFLOP/s")
            if "dram read" in cur and "dram write" in cur:
                out.append(f"- DRAM read+write: {(cur['dram read'] + cur['dram write']) / cur['duration'] / 1e9:.1f} GB/s")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    if kind == "rederive":
        print(rederive(path))
    else:
        print(full_report(path) if kind == "full" else launch_list(path))
