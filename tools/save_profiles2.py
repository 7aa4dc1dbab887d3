#!/usr/bin/env python
"""Round-2 tracked summaries under profiles/ from the scratch files of tools/gpu_prof2.sh (gpurun_out/)."""
import csv, json, subprocess, sys
from collections import defaultdict, Counter
tag = "r02"
# ---- launch list shares
rows = list(csv.reader(open('gpurun_out/r02_launches.csv')))
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
    val = val / 1e3 if unit in ('us', 'usecond') else val / 1e6 if unit in ('ns', 'nsecond') else val * 1e3 if unit in ('s', 'second') else val
    agg[name][0] += 1
    agg[name][1] += val
tot = sum(v[1] for v in agg.values())
lines = ["# ncu launch list (round 2)",
         "# command: ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 120 --csv python bench.py --iters 8 --steps 1 --warmup 3 --no-cpu-baseline",
         "# (116^3 cells Q5, the bench workload; the same command exited 0 without ncu immediately before).",
         "# Per-launch times are cold-cache and serialised: compare SHARES.  bench.py reports the share of the brick kernel",
         "# among the four iteration kernels live as roofline.kernel_share_of_step.",
         "kernel,launches,total_ms,share"]
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{k},{v[0]},{v[1]:.3f},{v[1] / tot:.3f}")
it = sum(agg[k][1] for k in agg if any(s in k for s in ('k_brick', 'k_pre', 'k_post', 'k_scalar_merged')))
br = sum(agg[k][1] for k in agg if 'k_brick' in k)
lines.append(f"# brick kernel share of the iteration kernels under ncu: {br / it:.3f}")
open(f'profiles/{tag}_launches.csv', 'w').write("\n".join(lines) + "\n")
print(lines[-1])
# ---- traffic
raw = list(csv.reader(subprocess.run(["ncu", "-i", "gpurun_out/prof_brick2.ncu-rep", "--page", "raw", "--csv"],
                                      capture_output=True, text=True).stdout.splitlines()))
h, u = raw[0], raw[1]
def val(r, k):
    i = h.index(k)
    return float(r[i].replace(',', '')) * {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1}.get(u[i], 1)
tr = [val(r, 'dram__bytes_read.sum') + val(r, 'dram__bytes_write.sum') for r in raw[2:]]
# (profiles/traffic.json is written from the 116^3 capture of tools/gpu_traffic116.sh; this 73^3 figure goes to the summary)
print("traffic B/DoF", [t / 49027896 for t in tr])
subprocess.run([sys.executable, "tools/ncu_summary.py", "gpurun_out/prof_brick2.ncu-rep", f"profiles/{tag}_ncu_brick2.txt",
                "k_brick2<5,double> (round 2); 73^3 cells Q5; ncu --set full --clock-control none --import-source on"],
               capture_output=True)
# ---- stall reasons per role (source page; role = range of source lines of mfcg_brick2.cuh)
out = subprocess.run(["ncu", "-i", "gpurun_out/prof_brick2.ncu-rep", "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:k_brick2"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = None; lines2 = []; nk = 0
for r in rows:
    if r and r[0] == "Line No":
        nk += 1
        if nk > 1: break
        hdr = r; continue
    if hdr and len(r) == len(hdr): lines2.append(r)
ix = {}
for i, k in enumerate(hdr): ix.setdefault(k, i)
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except ValueError: return 0.0
src = open('paper_2205_08909_b200/csrc/mfcg_brick2.cuh').read().splitlines()
def line_of(marker): return next(i + 1 for i, l in enumerate(src) if marker in l)
marks = [("producer", line_of("==== producer ====")), ("update", line_of("==== update warps ====")),
         ("plane sweeps", line_of("==== plane sweeps")), ("z sweep + gather", line_of("==== z sweep + gather")),
         ("end", line_of("// brick sums, fixed order") + 25)]
stalls = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
agg2 = {m[0]: Counter() for m in marks[:-1]}
cur = 0
for r in lines2:
    if not r[0].strip(): continue  # SASS rows repeat what their source row sums up
    try: cur = int(r[0])
    except ValueError: continue
    for (name, lo), (_, hi) in zip(marks[:-1], marks[1:]):
        if lo <= cur < hi:
            for s in stalls: agg2[name][s] += f(r, s)
            agg2[name]['inst'] += f(r, 'Instructions Executed')
with open(f'profiles/{tag}_ncu_brick2.txt', 'a') as fh:
    fh.write("warp-state samples per role (source lines of mfcg_brick2.cuh; first captured launch):\n")
    for name, c in agg2.items():
        t = sum(v for k, v in c.items() if k != 'inst')
        fh.write(f"  {name}: {c['inst'] / 1e6:.1f} M warp instructions, {int(t)} samples: " +
                 ' '.join(f"{k[6:]} {100 * v / t:.0f}%" for k, v in c.most_common() if k != 'inst' and v / t > 0.02) + "\n")
print(open(f'profiles/{tag}_ncu_brick2.txt').read()[-1500:])
