timeout 600 python -m pytest tests/test_boundary_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2v_tests.txt
timeout 900 python bench.py --steps 5 > gpurun_out/r2v_c5.json 2> gpurun_out/r2v_c5.err
LG=30; TAG=r2v
for spec in "lx_main 1 bwd" "lx_main 0 fwd" "lx_gather_agg 1 agg"; do
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
cat gpurun_out/r2v_tests.txt
python -c "
import json; d=json.load(open('gpurun_out/r2v_c5.json')); print('C5', round(d['ms_per_step'],3), d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'])
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step']): print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"
