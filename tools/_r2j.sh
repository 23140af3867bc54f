timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_boundary_gpu.py tests/test_acceptance_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2j_tests.txt
timeout 900 python -m pytest tests/test_parity_scale_gpu.py -x -q -k "c2 or c3 or c4" 2>&1 | tail -4 >> gpurun_out/r2j_tests.txt
for c in C2 C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2j_$c.json 2> gpurun_out/r2j_$c.err; done
cat gpurun_out/r2j_tests.txt
for c in C2 C3 C4 C5; do python -c "
import json; d=json.load(open('gpurun_out/r2j_$c.json')); print('$c', round(d['ms_per_step'],3))
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step'])[:6]: print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"; done
