#!/bin/bash
for lib in tools/varlibs/*.so; do cp $lib paper_2205_08909_b200/libmfcg_b200.so
for v in ${VARIANTS:-final_tensor_load inverse_jacobian_load}; do
python bench.py --cells 96 96 96 --geometry $v --deform 0.1 --iters 30 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib $v value %.3e kernel_ms %.3f it_ms %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms']))"
done; done
