timeout 900 python -m pytest tests/test_sharded_gpu.py tests/test_boundary_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/r2e_tests.txt
for c in C2 C3 C4 C5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2e_$c.json 2> gpurun_out/r2e_$c.err; done
for f in gpurun_out/r2e_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), 'dom', d['roofline']['kernel'], d['roofline']['frac'])"; done
cat gpurun_out/r2e_tests.txt
