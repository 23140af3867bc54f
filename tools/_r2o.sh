# ncu captures at 2^30: new sort pass, main bwd (source-level), perm scatter
LG=30; TAG=r2o
for spec in "lx_sort_pass 2 sort" "lx_main 1 bwd" "lx_main 0 fwd"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$1\$" -s $2 -c 1 \
      -o gpurun_out/${TAG}_$3 python tools/prof_step.py $LG 1 > gpurun_out/${TAG}_$3.log 2>&1
done
python tools/ncu_summary.py gpurun_out/${TAG}_*.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
for f in gpurun_out/${TAG}_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source cuda > $b.cuda.csv 2>/dev/null || true
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv $b.cuda.csv
  rm -f $f
done
cat gpurun_out/${TAG}_summary.txt; du -sh gpurun_out
