for v in g3 hoist agg2 agg8 agg2t128; do
  echo "== $v" >> gpurun_out/r2w_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|gather_agg|main_" >> gpurun_out/r2w_kt.txt
done
cat gpurun_out/r2w_kt.txt
