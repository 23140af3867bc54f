#!/bin/bash
# One profiling call: the launch list of one C5 step at 2^LG (time + DRAM bytes per launch)
# and ncu --set full captures of the main kernels, a mid sort pass and one gather+aggregate
# pass at the same size.  Numbers taken under ncu are never bench values.
LG=${1:-30}; TAG=${2:-r01m}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/prof_step.py $LG 1 > /dev/null 2>&1
for spec in "lx_main 0 fwd" "lx_main 1 bwd" "lx_sort_pass 2 sort" "lx_gather_agg 2 agg"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$1\$" -s $2 -c 1 \
      -o gpurun_out/${TAG}_$3 python tools/prof_step.py $LG 1 > gpurun_out/${TAG}_$3.log 2>&1
done

# export on the box (full reports at 2^30 exceed the copy-back limit); keep the csv pages
for f in gpurun_out/${TAG}_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $f
done
du -sh gpurun_out
