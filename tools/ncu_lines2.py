#!/usr/bin/env python
"""Per CUDA source line of the first captured kernel matching a regex: warp instructions, stall samples by
reason, shared-memory wavefronts.  usage: ncu_lines2.py report.ncu-rep kernel_regex [top]"""
import csv, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None; lines = []; nk = 0
for r in rows:
    if r and r[0] == "Line No":
        nk += 1
        if nk > 1: break
        hdr = r; continue
    if hdr and len(r) == len(hdr): lines.append(r)
ix = {}
for i, k in enumerate(hdr): ix.setdefault(k, i)
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except ValueError: return 0.0
agg = collections.defaultdict(lambda: collections.Counter()); text = {}
cur = None
for r in lines:
    # cuda,sass view: a source line row followed by its SASS rows (Line No empty?)  -- aggregate on the last seen source line
    if r[0].strip():
        cur = r[0].strip(); text.setdefault(cur, r[1].strip())
    a = agg[cur]
    a["inst"] += f(r, "Instructions Executed"); a["samp"] += f(r, "# Samples")
    a["smem"] += f(r, "L1 Wavefronts Shared"); a["smem_x"] += f(r, "L1 Wavefronts Shared Excessive")
    for k in ("stall_long_sb", "stall_barrier", "stall_short_sb", "stall_wait", "stall_math", "stall_mio", "stall_sleep", "stall_selected", "stall_no_inst"):
        a[k] += f(r, k)
ti = sum(a["inst"] for a in agg.values()); ts = sum(a["samp"] for a in agg.values()); tw = sum(a["smem"] for a in agg.values())
print(f"total warp inst {ti/1e6:.1f} M, samples {ts:.0f}, smem wavefronts {tw/1e6:.1f} M (excessive {sum(a['smem_x'] for a in agg.values())/1e6:.1f} M)")
for key in ("samp", "smem", "inst"):
    print(f"--- top by {key}")
    for ln, a in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"{ln:>5} inst {a['inst']/1e6:7.2f}M samp {100*a['samp']/ts:5.1f}% smem {a['smem']/1e6:6.2f}M(+{a['smem_x']/1e6:5.2f}) "
              f"lsb {a['stall_long_sb']:.0f} bar {a['stall_barrier']:.0f} ssb {a['stall_short_sb']:.0f} wait {a['stall_wait']:.0f} math {a['stall_math']:.0f} slp {a['stall_sleep']:.0f} | {text[ln][:80]}")
