#!/bin/bash
# full round-end style pass: tests, smoke, default bench (116^3), reference arm, ncu launch list + full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; grep -E '^E  |FAILED|passed|failed' gpurun_out/pytest_gpu.log | head
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -2 gpurun_out/bench_default.err
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -2 gpurun_out/bench_reference.err
lscpu | head -20 > gpurun_out/lscpu_box.txt
CMD="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
# the full capture of the brick kernel is a separate call: tools/gpu_prof.sh ncu
python bench.py --cells 73 73 73 --components 3 --steps 2 --no-cpu-baseline > gpurun_out/bench_bp4type_73.json 2> gpurun_out/bench_bp4.err; tail -2 gpurun_out/bench_bp4.err
