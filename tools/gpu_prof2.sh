#!/bin/bash
# one full ncu capture of the persistent brick kernel (73^3 cells, short solve)
mkdir -p gpurun_out
CMD="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_brick2 -s 12 -c 2 -o gpurun_out/prof_brick2 -f $CMD > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu2.log
