#!/bin/bash
# first measurement pass: bench at three sizes + ncu launch list + one full capture
set -x
mkdir -p gpurun_out
python bench.py --cells 48 48 48 --steps 2 --warmup 1 > gpurun_out/bench_48.json 2> gpurun_out/bench_48.err; tail -3 gpurun_out/bench_48.err
python bench.py --cells 73 73 73 > gpurun_out/bench_73.json 2> gpurun_out/bench_73.err; tail -3 gpurun_out/bench_73.err
python bench.py > gpurun_out/bench_116.json 2> gpurun_out/bench_116.err; tail -3 gpurun_out/bench_116.err
CMD="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_brick -s 3 -c 2 -o gpurun_out/prof_brick $CMD > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
