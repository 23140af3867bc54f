timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2d_c5.json 2> gpurun_out/r2d_c5.err
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2d_$c.json 2> gpurun_out/r2d_$c.err; done
timeout 900 python -m pytest tests/test_boundary_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/r2d_boundary.txt
for f in gpurun_out/r2d_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'][:40], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), 'dom', d['roofline']['kernel'], d['roofline']['frac'])"; done
cat gpurun_out/r2d_boundary.txt
