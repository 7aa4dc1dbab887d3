#!/usr/bin/env python
"""Per CUDA source line: warp instructions executed and stall samples of the first captured k_brick launch."""
import csv, subprocess, sys
rep = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_brick.ncu-rep"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:k_brick"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None; lines = []; seen_kernel = 0
for r in rows:
    if r and r[0] == "Function Name":
        seen_kernel += 1
        if seen_kernel > 1 and lines: break
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "Line No"):
        lines.append(r)
ix = {k: i for i, k in enumerate(hdr)}
src_i = 1
tot_i = sum(float(r[ix["Instructions Executed"]] or 0) for r in lines)
tot_s = sum(float(r[ix["# Samples"]] or 0) for r in lines)
print(f"total warp instructions {tot_i/1e6:.1f} M, samples {tot_s:.0f}")
lines.sort(key=lambda r: -float(r[ix["Instructions Executed"]] or 0))
for r in lines[:top]:
    print(f"{r[0]:>5} {float(r[ix['Instructions Executed']])/1e6:8.2f}M {100*float(r[ix['Instructions Executed']])/tot_i:5.1f}% samp {100*float(r[ix['# Samples']])/tot_s:5.1f}%  {r[src_i].strip()[:110]}")
