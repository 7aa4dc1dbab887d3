#!/bin/bash
run() { python bench.py --degree $1 --cells $2 $2 $2 --brick $3 $4 $5 --iters 50 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('p$1 brick $3x$4x$5 value %.3e kernel_ms %.3f it_ms %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms']))"; }
for bz in 16 32 64 128; do run 1 367 16 16 $bz; done
for bz in 16 32 64; do run 2 184 8 8 $bz; done
for bz in 16 32 48; do run 3 122 8 4 $bz; done
for bz in 16 24 32; do run 4 92 4 4 $bz; done
