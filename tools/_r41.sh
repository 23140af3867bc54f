for v in agg5 b3; do
  echo "== $v" >> gpurun_out/r41_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|gather_agg|main_" >> gpurun_out/r41_kt.txt
done
for v in agg5 b3; do
  for c in C2 C3; do
    LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r41_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r41_${v}_$c.json')); k=d['kernels']
print('$v $c', round(d['ms_per_step'],3), {n: k[n]['ms_per_step'] for n in k if n.startswith('lx_main') or n=='lx_gather_agg'})" >> gpurun_out/r41_kt.txt
  done
done
cat gpurun_out/r41_kt.txt
