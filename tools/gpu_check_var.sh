#!/bin/bash
# quick correctness (parity subset + ragged stress) of the production build, then the sustained 116^3 comparison of
# production and every tools/varlibs/*.so except timing.so, then the phase clocks of timing.so if present
timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ragged or q5 or midsize" 2>&1 | tail -2
timeout 200 python tools/stress.py 49 49 20 200 300 2>&1 | tail -1
mkdir -p /tmp/tv; mv tools/varlibs/timing.so /tmp/tv/ 2>/dev/null
bash tools/gpu_var116s.sh
if [ -f /tmp/tv/timing.so ]; then mkdir -p /tmp/tv2; mv tools/varlibs/*.so /tmp/tv2/ 2>/dev/null; mv /tmp/tv/timing.so tools/varlibs/; bash tools/gpu_timing116.sh; fi
