for v in sc1 bst2; do
  echo "== $v" >> gpurun_out/r46_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|perm_|main_" >> gpurun_out/r46_kt.txt
done
for c in C2 C3; do
  LAPLEX_LIB=$PWD/variants/lib_bst2.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r46_bst2_$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r46_bst2_$c.json')); k=d['kernels']
print('bst2 $c', round(d['ms_per_step'],3), {n: k[n]['ms_per_step'] for n in k if n.startswith('lx_perm') or n.startswith('lx_main')})" >> gpurun_out/r46_kt.txt
done
LAPLEX_LIB=$PWD/variants/lib_bst2.so timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_parity_scale_gpu.py tests/test_boundary_gpu.py -x -q 2>&1 | tail -3 >> gpurun_out/r46_kt.txt
cat gpurun_out/r46_kt.txt
