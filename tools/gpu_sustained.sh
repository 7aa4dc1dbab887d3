#!/bin/bash
# A/B under sustained load (the default bench: 116^3, 200 iterations per step): the B200 is power
# capped there, so energy per DoF counts as well as time at full clocks
for rep in 1 2; do
for lib in tools/varlibs/*.so; do cp $lib paper_2205_08909_b200/libmfcg_b200.so
python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$lib value %.3e kernel_ms %.3f it_ms %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
