echo "== g3" >> gpurun_out/r2t_kt.txt
LAPLEX_LIB=$PWD/variants/lib_g3.so timeout 300 python tools/kern_times.py 30 >> gpurun_out/r2t_kt.txt 2>&1
LAPLEX_LIB=$PWD/variants/lib_g3.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/r2t_tests.txt
./tools/perm_micro 30 2>&1 | grep -v "^window" > gpurun_out/r2t_micro.txt
cat gpurun_out/r2t_kt.txt gpurun_out/r2t_tests.txt gpurun_out/r2t_micro.txt
