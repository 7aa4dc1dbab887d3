#!/bin/bash
# timing experiments with phases disabled (results are wrong on purpose)
for lib in tools/varlibs/*.so; do
  cp $lib paper_2205_08909_b200/libmfcg_b200.so
  python bench.py --cells 73 73 73 --iters 20 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib', 'kernel_ms %.3f it_ms %.3f'%(r['kernel_ms'], r['iteration_ms']))"
done
