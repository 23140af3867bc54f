for v in cur h1 h8; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r44_sort.txt 2>&1
done
cat gpurun_out/r44_sort.txt
