#!/bin/bash
# production-flag variants at the bench workload under sustained load (116^3, 200 iterations per solve)
shopt -s nullglob
for lib in "" tools/varlibs/*.so; do
  MFCG_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-production}', 'value %.3e kernel_ms %.3f it_ms %.3f frac %.3f itfrac %.3f'%(d['value'], r['kernel_ms'], r['iteration_ms'], r['frac'], r['iteration_frac']), d['clocks']['sm_mhz'], d['extra']['brick'])"
done
