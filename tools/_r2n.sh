# sort ranking rewrite (sortA) vs base; permutation window/cache-policy micro
./tools/perm_micro 30 > gpurun_out/r2n_perm_micro.txt 2>&1
for v in base sortA base sortA; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r2n_sort.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_sortA.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q -k "sort or perm or coranks or golden or plan" 2>&1 | tail -4 > gpurun_out/r2n_tests.txt
cat gpurun_out/r2n_perm_micro.txt gpurun_out/r2n_sort.txt gpurun_out/r2n_tests.txt
