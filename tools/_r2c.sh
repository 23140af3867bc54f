timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_parity_scale_gpu.py::test_c5_full_size_2p30 --deselect "tests/test_parity_scale_gpu.py::test_c5_shape_fwd_bwd_against_oracle[28]" 2>&1 | tail -15 > gpurun_out/r2c_pytest.txt
timeout 1200 python -m pytest tests/test_parity_scale_gpu.py -x -q -s --durations=0 -k "c2 or c3 or c4" 2>&1 | tail -30 > gpurun_out/r2c_cfg.txt
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
cat gpurun_out/r2c_pytest.txt gpurun_out/r2c_cfg.txt; tail -c 600 gpurun_out/r2c_bench.json
