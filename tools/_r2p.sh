for v in sortA sortB sortB3 sortB; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r2p_sort.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_sortB.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q -k "sort or perm or coranks or golden or plan" 2>&1 | tail -4 > gpurun_out/r2p_tests.txt
cat gpurun_out/r2p_sort.txt gpurun_out/r2p_tests.txt
