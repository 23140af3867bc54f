for v in mw ps; do
  echo "== $v" >> gpurun_out/r2r_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 >> gpurun_out/r2r_kt.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_ps.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2r_tests.txt
cat gpurun_out/r2r_kt.txt gpurun_out/r2r_tests.txt
