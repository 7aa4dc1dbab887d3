#!/bin/bash
cells=(0 367 184 122 92 73 61 52 46)
for lib in tools/varlibs/*.so; do cp $lib paper_2205_08909_b200/libmfcg_b200.so
for p in $DEGS; do n=${cells[$p]}
python bench.py --degree $p --cells $n $n $n --iters 50 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib p$p value %.3e kernel_ms %.3f it_ms %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms']))"
done; done
