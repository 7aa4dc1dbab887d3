#!/bin/bash
# round 2 evidence: plain run, launch list of the bench command, one full ncu capture of the persistent brick kernel
mkdir -p gpurun_out
CMD="python bench.py --iters 8 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 120 --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu1.log 2>&1
tail -2 gpurun_out/ncu1.log
CMD2="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_brick2 -s 12 -c 2 -o gpurun_out/prof_brick2 -f $CMD2 > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
