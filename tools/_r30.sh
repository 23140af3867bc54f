for c in C2 C3 C4 C1; do
  timeout 900 python bench.py --config $c > gpurun_out/r30_bench_$c.json 2> gpurun_out/r30_bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^lx_main\$" -s 1 -c 1 \
    -o gpurun_out/r30_c2bwd python bench.py --config C2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r30_c2bwd.log 2>&1
python tools/ncu_summary.py gpurun_out/r30_c2bwd.ncu-rep > gpurun_out/r30_c2bwd_summary.txt 2>&1
ncu -i gpurun_out/r30_c2bwd.ncu-rep --page source --csv --print-source sass > gpurun_out/r30_c2bwd.sass.csv 2>/dev/null; gzip -f gpurun_out/r30_c2bwd.sass.csv
ncu -i gpurun_out/r30_c2bwd.ncu-rep --page raw --csv > gpurun_out/r30_c2bwd.raw.csv 2>/dev/null
rm -f gpurun_out/r30_c2bwd.ncu-rep
for c in C1 C2 C3 C4; do python -c "
import json; d=json.load(open('gpurun_out/r30_bench_$c.json')); print('$c', round(d['ms_per_step'],3), d['value'], d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['ms_per_step'] if d.get('e2e') else None)
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:8]: print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"; done
cat gpurun_out/r30_c2bwd_summary.txt | head -30
