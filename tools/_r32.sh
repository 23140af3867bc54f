LG=30; TAG=r32
for spec in "lx_group_plan 0 gplan" "lx_sort_pass 8 splan"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$1\$" -s $2 -c 1 \
      -o gpurun_out/${TAG}_$3 python tools/prof_step.py $LG 1 > gpurun_out/${TAG}_$3.log 2>&1
done
python tools/ncu_summary.py gpurun_out/${TAG}_*.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
for f in gpurun_out/${TAG}_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
  rm -f $f
done
cat gpurun_out/${TAG}_summary.txt
