#!/bin/bash
# DRAM traffic of the brick kernel at the bench workload itself (116^3 cells Q5): two consecutive launches, one with
# and one without the x update.  Plain run first, then the same command under ncu (three metrics, no full set).
mkdir -p gpurun_out
CMD="python bench.py --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain116.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_brick2 -s 12 -c 2 \
    --csv --log-file gpurun_out/r02_traffic116.csv $CMD > gpurun_out/ncu116.log 2>&1
tail -2 gpurun_out/ncu116.log; tail -8 gpurun_out/r02_traffic116.csv
