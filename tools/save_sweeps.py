#!/usr/bin/env python
"""gpurun_out/sw_*.json (tools/gpu_sweep.sh) -> profiles/<tag>_sweeps.csv"""
import glob, json, os, sys
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for f in sorted(glob.glob("gpurun_out/sw_*.json")):
    try:
        d = json.load(open(f))
    except Exception:
        continue
    c, r = d["config"], d["roofline"]
    name = os.path.basename(f)[3:-5]
    info = d.get("extra", {})
    rows.append([name, c["degree"], c["cells"][0], c["n_dofs"], c["variant"], d["dtype"], f"{d['value']:.4g}",
                 f"{d['e2e']['value']:.4g}", f"{r['kernel_ms']:.4g}", f"{r['iteration_ms']:.4g}",
                 f"{r['iteration_frac']:.4g}", "x".join(str(b) for b in info.get("brick", [])),
                 f"{info.get('final_relative_residual', float('nan')):.4g}"])
out = f"profiles/{tag}_sweeps.csv"
with open(out, "w") as fh:
    fh.write("# Sweeps on one B200 (tools/gpu_sweep.sh; 50 fixed iterations per solve, 2 timed solves, ladder: 200 iterations)\n"
             "# BASELINE configs[3]: degree sweep at ~5e7 DoFs, fp64 and fp32, merged (combined_pcg) vs standard (pcg);\n"
             "# BASELINE configs[1]: size ladder Q5; plus brick depth Bz at 73^3.  iteration_frac = 64 B (32 B fp32) x n_dofs / iteration time / 6551 GB/s.\n"
             "tag,degree,cells_per_dim,n_dofs,variant,dtype,DoF_it_per_s,e2e_DoF_it_per_s,operator_kernel_ms,iteration_ms,iteration_frac,brick,final_rel_residual\n")
    for r in rows:
        fh.write(",".join(str(x) for x in r) + "\n")
print(out, len(rows))
