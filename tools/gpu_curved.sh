#!/bin/bash
# BASELINE configs[2]: 96^3 cells Q5 on the sine-deformed mesh (amplitude 0.1), stored vs on-the-fly geometry
mkdir -p gpurun_out
for v in final_tensor_load inverse_jacobian_load quadratic_compute; do
python bench.py --cells 96 96 96 --geometry $v --deform 0.1 --iters 50 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/curved96_$v.json 2> gpurun_out/curved96_$v.err || tail -2 gpurun_out/curved96_$v.err
python -c "
import json; d=json.load(open('gpurun_out/curved96_$v.json')); r=d['roofline']; print('$v value %.3e kernel_ms %.3f it_ms %.3f frac %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms'], r['frac']))"
done
