timeout 2400 python -m pytest tests/test_parity_scale_gpu.py -x -q -s --durations=0 2>&1 | tail -40 > gpurun_out/r2b_pytest.txt
cat gpurun_out/r2b_pytest.txt
