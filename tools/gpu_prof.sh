#!/bin/bash
# ncu captures for one step at 2^LG (run under gpurun; numbers are never bench values)
LG=${1:-28}
TAG=${2:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/prof_step.py $LG 1 > /dev/null 2>&1
for K in lx_sort_pass lx_perm_scatter lx_fix_fwd lx_main_bwd lx_main_fwd lx_fix_bwd lx_splan lx_perm_gather; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/${TAG}_$K python tools/prof_step.py $LG 1 > gpurun_out/${TAG}_$K.log 2>&1
done
ls -la gpurun_out
