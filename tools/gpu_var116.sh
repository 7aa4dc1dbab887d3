#!/bin/bash
# production-flag variants at the bench workload (116^3, short solves); extra args go to bench.py
for lib in tools/varlibs/*.so; do
  MFCG_LIB=$PWD/$lib timeout 200 python bench.py --iters 50 --steps 2 --warmup 2 --no-cpu-baseline "$@" 2>gpurun_out/$(basename $lib).err | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', 'value %.3e kernel_ms %.3f it_ms %.3f frac %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms'], r['frac']), d['clocks']['sm_mhz'], d['extra']['brick'])"
done
