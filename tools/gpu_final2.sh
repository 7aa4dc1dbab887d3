#!/bin/bash
# round-2 record: GPU tests, the default bench (both arms), launch list + full ncu capture of the brick kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02_pytest_gpu.log
lscpu > gpurun_out/r02_lscpu_box.txt
python bench.py > gpurun_out/r02_bench_116.json 2> gpurun_out/r02_bench_116.err; tail -2 gpurun_out/r02_bench_116.err
python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_ref.err; tail -2 gpurun_out/r02_bench_ref.err
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_116.json')); r=d['roofline']; print('value %.3e e2e %.3e kernel_ms %.3f it_ms %.3f frac %.3f it_frac %.3f cpu %.3e'%(d['value'], d['e2e']['value'], r['kernel_ms'], r['iteration_ms'], r['frac'], r['iteration_frac'], d['cpu_baseline']['value']), d['clocks'])
d=json.load(open('gpurun_out/r02_bench_reference_arm.json')); print('reference arm %.3e'%d['value'], d['config']['workload'])"
bash tools/gpu_prof2.sh
