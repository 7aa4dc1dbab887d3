#!/bin/bash
# ncu counters of the brick kernel for every library in tools/varlibs (one ncu pass per library is
# not allowed in one call: this script takes the library name as $1)
lib=$1
cp tools/varlibs/$lib paper_2205_08909_b200/libmfcg_b200.so
CMD="python bench.py --cells 73 73 73 --iters 8 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum \
  --clock-control none -k regex:k_brick -s 3 -c 2 --csv --log-file gpurun_out/metrics_$lib.csv $CMD > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/metrics_$lib.csv')))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hd=rows[h]; n=hd.index('Metric Name'); v=hd.index('Metric Value'); u=hd.index('Metric Unit'); idc=hd.index('ID')
for r in rows[h+1:]:
    if len(r)>v: print(r[idc], r[n], r[v], r[u])
PY
