for v in ilp ilp3; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r2u_sort.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_ilp.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_boundary_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2u_tests.txt
cat gpurun_out/r2u_sort.txt gpurun_out/r2u_tests.txt
