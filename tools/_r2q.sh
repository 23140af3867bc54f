for v in sortB mw; do
  echo "== $v" >> gpurun_out/r2q_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 >> gpurun_out/r2q_kt.txt 2>&1
done
LAPLEX_LIB=$PWD/variants/lib_mw.so timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_parity_scale_gpu.py tests/test_sharded_gpu.py tests/test_acceptance_gpu.py tests/test_density_gpu.py -x -q 2>&1 | tail -6 > gpurun_out/r2q_tests.txt
cat gpurun_out/r2q_kt.txt gpurun_out/r2q_tests.txt
