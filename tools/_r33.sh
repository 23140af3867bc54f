for v in gp3; do
  echo "== $v" >> gpurun_out/r33_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 >> gpurun_out/r33_kt.txt
done
LAPLEX_LIB=$PWD/variants/lib_gp3.so timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_parity_scale_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r33_tests.txt
cat gpurun_out/r33_kt.txt gpurun_out/r33_tests.txt
