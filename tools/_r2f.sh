timeout 1200 python -m pytest tests/test_sanitizer_gpu.py -x -q 2>&1 | tail -15 > gpurun_out/r2f_san.txt
timeout 600 python bench.py --sim 2 --log2n 26 --steps 3 > gpurun_out/r2f_sim2.json 2> gpurun_out/r2f_sim2.err
timeout 600 python bench.py --sim 8 --log2n 27 --steps 3 > gpurun_out/r2f_sim8.json 2> gpurun_out/r2f_sim8.err
timeout 900 python bench.py > gpurun_out/r2f_c5.json 2> gpurun_out/r2f_c5.err
timeout 900 python bench.py --impl reference > gpurun_out/r2f_ref_c5.json 2> gpurun_out/r2f_ref_c5.err
cat gpurun_out/r2f_san.txt; tail -c 400 gpurun_out/r2f_sim2.json; tail -c 400 gpurun_out/r2f_sim8.json; tail -5 gpurun_out/r2f_sim8.err
python -c "
import json; d=json.load(open('gpurun_out/r2f_c5.json')); print(d['ms_per_step'], d['cpu_baseline']); r=json.load(open('gpurun_out/r2f_ref_c5.json')); print(r['value'], r['ms_per_step'], r['cpu_baseline']['sample'])"
