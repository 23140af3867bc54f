timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r39_c5.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r39_c5.json')); print('C5', round(d['ms_per_step'],3), d['roofline']['frac'])
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step']): print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
