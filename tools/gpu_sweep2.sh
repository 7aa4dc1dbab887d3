#!/bin/bash
# round 2: degree sweep at ~5e7 DoFs (fp64 merged with the persistent kernel on/off, standard PCG, fp32), size ladder,
# 3 components, curved 96^3; results as one line per run in gpurun_out/r02_sweeps.txt
mkdir -p gpurun_out
out=gpurun_out/r02_sweeps.txt; : > $out
run() { tag=$1; shift; timeout 300 python bench.py --steps 2 --warmup 1 --iters 50 --no-cpu-baseline "$@" > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err || tail -2 gpurun_out/sw_$tag.err; python - <<PY | tee -a $out
import json
try:
    d=json.load(open("gpurun_out/sw_$tag.json")); r=d["roofline"]
    print("$tag value %.3e e2e %.3e kernel_ms %.3f it_ms %.3f kfrac %.3f it_frac %.3f res %.2e brick %s"%(d["value"],d["e2e"]["value"],r["kernel_ms"],r["iteration_ms"],r["frac"],r["iteration_frac"],d["extra"]["final_relative_residual"],d["extra"]["brick"]))
except Exception as e: print("$tag failed", e)
PY
}
cells=(0 367 184 122 92 73 61 52 46)
for p in ${DEGS:-1 2 3 4 5 6 7 8}; do n=${cells[$p]}
  run p${p}_f64_merged --degree $p --cells $n $n $n
  MFCG_BRICK2=0 run p${p}_f64_merged_gen1 --degree $p --cells $n $n $n
  run p${p}_f64_pcg --degree $p --cells $n $n $n --variant pcg
  run p${p}_f32_merged --degree $p --cells $n $n $n --precision fp32
done
if [ -z "$NOEXTRA" ]; then
for n in 8 16 32 48 64 80 96; do run ladder$n --cells $n $n $n --iters 200; done
run bp4type_73 --cells 73 73 73 --components 3
for v in final_tensor_load inverse_jacobian_load quadratic_compute; do run curved96_$v --cells 96 96 96 --deform 0.1 --geometry $v; done
fi
