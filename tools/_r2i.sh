for v in 3_2 2_2 2_1 1_1; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/r2i_C3_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r2i_C3_$v.json')); print('$v', round(d['ms_per_step'],3), {k: v['ms_per_step'] for k,v in d['kernels'].items() if 'main' in k or 'agg' in k})"
done
