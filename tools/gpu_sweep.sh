#!/bin/bash
# BASELINE configs[3]/[1]: degree sweep at ~5e7 DoFs (fp64 + fp32, merged vs standard), size ladder, brick depth
mkdir -p gpurun_out
run() { tag=$1; shift; python bench.py --steps 2 --warmup 1 --iters 50 --no-cpu-baseline "$@" > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err || tail -2 gpurun_out/sw_$tag.err; python - <<PY
import json
try:
    d=json.load(open("gpurun_out/sw_$tag.json")); r=d["roofline"]
    print("$tag value %.3e e2e %.3e kernel_ms %.3f it_ms %.3f it_frac %.3f res %.2e"%(d["value"],d["e2e"]["value"],r["kernel_ms"],r["iteration_ms"],r["iteration_frac"],d["extra"]["final_relative_residual"]))
except Exception as e: print("$tag failed", e)
PY
}
for bz in 4 12 16 24; do run bz$bz --cells 73 73 73 --brick 4 4 $bz; done
cells=(0 367 184 122 92 73 61 52 46)
for p in 1 2 3 4 5 6 7 8; do n=${cells[$p]}; run p${p}_f64_merged --degree $p --cells $n $n $n; run p${p}_f64_pcg --degree $p --cells $n $n $n --variant pcg; run p${p}_f32_merged --degree $p --cells $n $n $n --precision fp32; done
for n in 4 8 16 32 48 64 96; do run ladder$n --cells $n $n $n --iters 200; done
