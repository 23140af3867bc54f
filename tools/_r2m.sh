timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2m_tests.txt
timeout 600 python bench.py > gpurun_out/r2m_c5.json 2> gpurun_out/r2m_c5.err
cat gpurun_out/r2m_tests.txt
python -c "
import json; d=json.load(open('gpurun_out/r2m_c5.json')); print('C5', round(d['ms_per_step'],3), d['e2e'], d.get('clocks'))
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step']): print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"
