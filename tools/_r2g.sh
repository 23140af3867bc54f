timeout 1500 python -m pytest tests/test_sanitizer_gpu.py tests/test_boundary_gpu.py -q 2>&1 | tail -5 > gpurun_out/r2g_san.txt
for n in 4195304; do /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 4 tools/sanitize_driver $n 1 > gpurun_out/r2g_mc.txt 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2g_c5.json 2> gpurun_out/r2g_c5.err
for c in C2 C3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2g_$c.json 2> gpurun_out/r2g_$c.err; done
cat gpurun_out/r2g_san.txt; head -20 gpurun_out/r2g_mc.txt
for f in gpurun_out/r2g_c*.json gpurun_out/r2g_C*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2))"; done
