timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|perm_|main_|sort_hist" > gpurun_out/r47_kt.txt
for c in C2 C3; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/r47_$c.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r47_$c.json')); k=d['kernels']
print('$c', round(d['ms_per_step'],3), {n: k[n]['ms_per_step'] for n in k if n.startswith('lx_perm') or n.startswith('lx_main')})" >> gpurun_out/r47_kt.txt
done
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/r47_kt.txt
cat gpurun_out/r47_kt.txt
