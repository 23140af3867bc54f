for v in scatter_a scatter_b scatter_a scatter_b; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/r2l_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r2l_$v.json')); k=d['kernels']; print('$v', round(d['ms_per_step'],2), k['lx_perm_scatter']['ms_per_step'], k['lx_perm_gather']['ms_per_step'])"
done
