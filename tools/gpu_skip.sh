#!/bin/bash
# timing experiments with variant builds (tools/varlibs/*.so, built with
# `python -m paper_2205_08909_b200.build --variant tools/varlibs/<name>.so -D...`); the variant is loaded
# through MFCG_LIB, the production library stays untouched
for lib in tools/varlibs/*.so; do
  MFCG_LIB=$PWD/$lib timeout 100 python bench.py --cells 73 73 73 --iters 20 --steps 2 --warmup 1 --no-cpu-baseline 2>gpurun_out/$(basename $lib).err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', 'kernel_ms %.3f it_ms %.3f'%(r['kernel_ms'], r['iteration_ms']))"
  grep -A18 'mfcg timing' gpurun_out/$(basename $lib).err | tail -18 | awk '{printf "%s %.0f | ", $1, $2/2960/200} END {print ""}'
done
