#!/bin/bash
# tests + bench (73^3) + one full ncu capture of the brick kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; grep -E '^E  |FAILED|passed|failed' gpurun_out/pytest_gpu.log | head -12
python bench.py --cells 73 73 73 --no-cpu-baseline > gpurun_out/bench_73_cur.json 2>gpurun_out/err.log; tail -2 gpurun_out/err.log
python -c "
import json; d=json.load(open('gpurun_out/bench_73_cur.json')); r=d['roofline']; print('value %.3e kernel_ms %.3f it_ms %.3f frac %.3f it_frac %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms'], r['frac'], r['iteration_frac']), d['clocks'])"
if [ "$1" = "ncu" ]; then
CMD="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_brick -s 3 -c 2 -o gpurun_out/prof_brick -f $CMD > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
fi
