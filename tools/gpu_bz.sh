#!/bin/bash
for bz in 16 20 24 29 39 58; do
python bench.py --brick 4 4 $bz --iters 50 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bz $bz value %.3e kernel_ms %.3f it_ms %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms']))"
done
