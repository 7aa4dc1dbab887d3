#!/usr/bin/env python
"""Turn the scratch files of tools/gpu_full.sh (gpurun_out/) into the tracked summaries under profiles/."""
import csv, json, subprocess, sys, shutil
from collections import defaultdict
tag = sys.argv[1] if len(sys.argv) > 1 else "r01_final"
rows = list(csv.reader(open('gpurun_out/launches.csv')))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
idx = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) < len(hdr):
        continue
    name = r[idx["Kernel Name"]].split('(')[0]
    val = float(r[idx["Metric Value"]].replace(',', ''))
    unit = r[idx["Metric Unit"]]
    val = val / 1e3 if unit == 'us' else val / 1e6 if unit == 'ns' else val * 1e3 if unit == 's' else val
    agg[name][0] += 1
    agg[name][1] += val
tot = sum(v[1] for v in agg.values())
lines = [f"# ncu launch list ({tag})",
         "# command: ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 3 --no-cpu-baseline",
         "# (the same command exited 0 without ncu immediately before).  Per-launch times are cold-cache and serialised: compare SHARES.",
         "# Set-up kernels (k_build_perm, k_diag_*, permutations) run once per operator / solve; bench.py reports the share of",
         "# k_brick among the four iteration kernels live as roofline.kernel_share_of_step.",
         "kernel,launches,total_ms,share"]
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{v[0]},{v[1]:.3f},{v[1] / tot:.3f}")
it = sum(agg[k][1] for k in agg if any(s in k for s in ('k_brick', 'k_pre', 'k_post', 'k_scalar_merged')))
br = sum(agg[k][1] for k in agg if 'k_brick' in k)
lines.append(f"# k_brick share of the iteration kernels under ncu: {br / it:.3f}")
open(f'profiles/{tag}_launches.csv', 'w').write("\n".join(lines) + "\n")
print(lines[-1])
raw = list(csv.reader(subprocess.run(["ncu", "-i", "gpurun_out/prof_brick.ncu-rep", "--page", "raw", "--csv"],
                                      capture_output=True, text=True).stdout.splitlines()))
h, u = raw[0], raw[1]
def val(r, k):
    i = h.index(k)
    return float(r[i].replace(',', '')) * {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}.get(u[i], 1)
tr = [val(r, 'dram__bytes_read.sum') + val(r, 'dram__bytes_write.sum') for r in raw[2:]]
json.dump({"k_brick_merged_bytes_per_launch": sum(tr) / len(tr), "launches": tr,
           "workload": "73^3 cells Q5 (49027896 DoFs)", "bytes_per_dof": sum(tr) / len(tr) / 49027896,
           "source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum, two consecutive launches "
                     "(one with, one without the x update); model 64 / 48 B per DoF on interior DoFs (the separable 1/diag is computed, not loaded)"},
          open('profiles/traffic.json', 'w'), indent=1)
print("traffic B/DoF", [t / 49027896 for t in tr])
subprocess.run([sys.executable, "tools/ncu_summary.py", "gpurun_out/prof_brick.ncu-rep", f"profiles/{tag}_ncu_brick.txt",
                f"k_brick ({tag}); 73^3 cells Q5; ncu --set full --clock-control none --import-source on"],
               capture_output=True)
shutil.copy('gpurun_out/bench_default.json', f'profiles/{tag}_bench_116.json')
shutil.copy('gpurun_out/bench_reference.json', f'profiles/{tag}_bench_reference_arm.json')
shutil.copy('gpurun_out/lscpu_box.txt', f'profiles/{tag}_lscpu_box.txt')
d = json.load(open('gpurun_out/bench_default.json')); r = d['roofline']
print("value %.3e e2e %.3e kernel_ms %.3f it_ms %.3f frac %.3f it_frac %.3f traffic %s cpu %.3e" % (
    d['value'], d['e2e']['value'], r['kernel_ms'], r['iteration_ms'], r['frac'], r['iteration_frac'], r['traffic'], d['cpu_baseline']['value']))
