for v in cur agg3 agg4; do
  echo "== $v" >> gpurun_out/r40_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|gather_agg|main_" >> gpurun_out/r40_kt.txt
done
for v in cur agg4; do
  for c in C2 C3; do
    LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r40_${v}_$c.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/r40_${v}_$c.json')); k=d['kernels']
print('$v $c', round(d['ms_per_step'],3), k['lx_gather_agg']['ms_per_step'])" >> gpurun_out/r40_kt.txt
  done
done
cat gpurun_out/r40_kt.txt
