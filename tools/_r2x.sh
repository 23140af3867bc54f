for v in hoist2 b256 f256; do
  echo "== $v" >> gpurun_out/r2x_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|gather_agg|main_" >> gpurun_out/r2x_kt.txt
done
cat gpurun_out/r2x_kt.txt
