for v in it20 it24c3 it28c3 it32c3; do
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/sort_bench.py 30 $v >> gpurun_out/r38_sort.txt 2>&1
done
cat gpurun_out/r38_sort.txt
