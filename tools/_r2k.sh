timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_density_gpu.py tests/test_boundary_gpu.py tests/test_scale_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/r2k_tests.txt
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r2k_c5.json 2> gpurun_out/r2k_c5.err
timeout 600 python bench.py --sim 4 --log2n 26 --steps 3 > gpurun_out/r2k_sim4.json 2> gpurun_out/r2k_sim4.err
cat gpurun_out/r2k_tests.txt; tail -3 gpurun_out/r2k_sim4.err; tail -c 300 gpurun_out/r2k_sim4.json
python -c "
import json; d=json.load(open('gpurun_out/r2k_c5.json')); print('C5', round(d['ms_per_step'],3))
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['ms_per_step']): print('   ', k, v['ms_per_step'], v['launches_per_step'], v['achieved_gbs'])
"
