"""Summarise an ncu --set full report of one kernel: key throughput metrics,
stall reasons (sampling), top stalled SASS lines.  usage: ncu_summary.py REP"""
import csv, io, subprocess, sys

rep = sys.argv[1]
def page(p, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))
raw = page("raw")
h, v = raw[0], raw[2]
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
src = page("source", "--print-source", "sass")
hdr, data = src[1], src[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
ix = [hdr.index(c) for c in cols]
tot = sum(int(r[iS] or 0) for r in data)
st = {c[6:]: sum(int(r[i] or 0) for r in data) for c, i in zip(cols, ix)}
print("stall share:", ", ".join(f"{k} {v / tot:.3f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]))
ops = {}
for r in data:
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + int(r[iS] or 0)
print("samples by opcode:", ", ".join(f"{k} {v / tot:.3f}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:12]))
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]:
    top = {c[6:]: int(r[i]) for c, i in zip(cols, ix) if r[i] not in ("0", "") and int(r[i]) > 0.15 * int(r[iS])}
    print(f"  {r[0][-5:]} {r[1].strip()[:58]:58s} {int(r[iS]) / tot:.3f} {top}")
