for v in gp2; do
  echo "== $v" >> gpurun_out/r2s_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 >> gpurun_out/r2s_kt.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_gp2.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2s_tests.txt
cat gpurun_out/r2s_kt.txt gpurun_out/r2s_tests.txt
