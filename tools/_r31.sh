for v in cur cpf; do
  for c in C1 C2 C3 C4 C5; do
    LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r31_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r31_${v}_$c.json')); k=d['kernels']
print('$v $c', round(d['ms_per_step'],3), {n: k[n]['ms_per_step'] for n in k if n.startswith('lx_main') or n=='lx_sort_hist'})" >> gpurun_out/r31.txt
  done
done
LAPLEX_LIB=$PWD/variants/lib_cpf.so timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_parity_scale_gpu.py tests/test_boundary_gpu.py tests/test_sharded_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r31_tests.txt
cat gpurun_out/r31.txt gpurun_out/r31_tests.txt
