# One gpurun call that regenerates the round's evidence at HEAD (TAG below): bench lines
# (C5 default + C1..C4), the ncu launch list of the bench command with per-kernel DRAM traffic,
# and full ncu captures of the dominant kernels (summaries in profiles/).  Usage: bash tools/gpu_evidence.sh TAG
TAG=${1:-r02f}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.err
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches_n2p30.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches_n2p30.csv > gpurun_out/${TAG}_launches_n2p30_summary.txt 2>&1
python tools/traffic_json.py gpurun_out/${TAG}_launches_n2p30.csv 30 gpurun_out/${TAG}_traffic.json > /dev/null 2>&1
for spec in "lx_sort_pass 2 sort" "lx_perm_stage_scatter 0 scatter" "lx_main 1 bwd" "lx_gather_agg 1 agg"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$1\$" -s $2 -c 1 \
      -o gpurun_out/${TAG}_$3 python tools/prof_step.py 30 1 > gpurun_out/${TAG}_$3.log 2>&1
done
python tools/ncu_summary.py gpurun_out/${TAG}_*.ncu-rep > gpurun_out/${TAG}_ncu_full_n2p30.txt 2>&1
for f in gpurun_out/${TAG}_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  rm -f $f
done
cat gpurun_out/${TAG}_launches_n2p30_summary.txt | head -30
python -c "
import json
for c in ['C5','C1','C2','C3','C4']:
    d=json.load(open('gpurun_out/${TAG}_bench_%s.json'%c)); print(c, round(d['ms_per_step'],3), '%.3g'%d['value'], d['roofline']['kernel'], d['roofline']['frac'], d.get('step_roofline',{}).get('frac'), d['e2e']['ms_per_step'] if d.get('e2e') else None, d.get('cpu_baseline',{}).get('value'), d.get('clocks'))
"
