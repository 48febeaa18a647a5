"""Copy the evidence of the last round-style GPU pass (gpurun_out/) into
profiles/<tag>_*: bench lines, config sweep, launch list + summary, ncu
metrics of the evaluator.  usage: update_profiles.py TAG"""
import json, os, shutil, subprocess, sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = "gpurun_out", "profiles"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


json.dump(last_json(f"{G}/bench.json"), open(f"{P}/{tag}_bench.json", "w"), indent=1)
json.dump(last_json(f"{G}/bench_ref.json"), open(f"{P}/{tag}_bench_reference.json", "w"), indent=1)
cfg = {}
for c in ("c1", "c3", "c4", "fast"):
    f = f"{G}/bench_{c}.json"
    if os.path.exists(f):
        cfg[c] = last_json(f)
json.dump(cfg, open(f"{P}/{tag}_bench_configs.json", "w"), indent=1)
shutil.copy(f"{G}/prof_launches.csv", f"{P}/{tag}_launches.csv")
out = subprocess.run([sys.executable, "scripts/summarize_launches.py", f"{P}/{tag}_launches.csv"],
                     capture_output=True, text=True).stdout
open(f"{P}/{tag}_launches_summary.txt", "w").write(out)
rep = os.path.join(ROOT, G, f"prof_eval_{tag}.ncu-rep")
summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "12"], capture_output=True,
                      text=True, cwd="/tmp").stdout
open(f"{P}/{tag}_eval_tc_ncu_summary.txt", "w").write(summ)
m = {}
for line in summ.splitlines():
    parts = line.split()
    if len(parts) == 2 and "__" in parts[0]:
        m[parts[0]] = float(parts[1])
json.dump({"kernel": "eval_tcs_kernel<18, 6, false, 4> (strict, streaming)", "frames_per_launch": 10,
           "dram_bytes_read": m.get("dram__bytes_read.sum", 0) * 1e6,
           "dram_bytes_write": m.get("dram__bytes_write.sum", 0) * 1e6,
           "duration_ms_under_ncu": m.get("gpu__time_duration.sum"),
           "xu_pct": m.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
           "issue_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "source": f"profiles/{tag}_eval_tc_ncu_summary.txt"},
          open(f"{P}/{tag}_eval_tc_ncu.json", "w"))
print(summ)
print(out)
