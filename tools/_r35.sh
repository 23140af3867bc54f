for v in offs; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r35_sort.txt 2>&1
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r35_sort.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_offs.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q -k "sort or perm or coranks or golden or plan" 2>&1 | tail -3 > gpurun_out/r35_tests.txt
cat gpurun_out/r35_sort.txt gpurun_out/r35_tests.txt
