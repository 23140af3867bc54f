for v in cur knob; do
  echo "== $v" >> gpurun_out/r43_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|perm_|sort_" >> gpurun_out/r43_kt.txt
  for c in C2 C3 C4; do
    LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r43_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r43_${v}_$c.json')); k=d['kernels']
print('$v $c', round(d['ms_per_step'],3), {n: k[n]['ms_per_step'] for n in k if n.startswith('lx_perm')})" >> gpurun_out/r43_kt.txt
  done
done
LAPLEX_LIB=$PWD/variants/lib_knob.so timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_boundary_gpu.py -x -q 2>&1 | tail -3 >> gpurun_out/r43_kt.txt
cat gpurun_out/r43_kt.txt
