for v in g3 cur; do
  echo "== $v" >> gpurun_out/r2y_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 >> gpurun_out/r2y_kt.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r2y_tests.txt
cat gpurun_out/r2y_kt.txt gpurun_out/r2y_tests.txt
