/usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 6 $PWD/tools/sanitize_driver 9000 2 > gpurun_out/r2h_ic.txt 2>&1
grep -v "Host Frame" gpurun_out/r2h_ic.txt | head -60
