#!/bin/bash
# per-role phase clocks of the persistent kernel at the bench workload (timing build, MFCG_LIB)
shopt -s nullglob
for lib in tools/varlibs/*.so; do
  MFCG_LIB=$PWD/$lib timeout 200 python bench.py --iters 20 --steps 2 --warmup 1 --no-cpu-baseline 2>gpurun_out/$(basename $lib).err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', 'kernel_ms %.3f it_ms %.3f'%(r['kernel_ms'], r['iteration_ms']), d['extra']['brick'])"
  # cycles per cell layer of one block: 20 launches per solve, 148 blocks, 3364 bricks x 29 layers / 148 blocks
  grep -A19 'mfcg timing' gpurun_out/$(basename $lib).err | tail -19 | awk '{printf "%s %.0f | ", $1, $2/20/148/659.1} END {print ""}'
done
