for v in cur sc2 ga32 agg512; do
  echo "== $v" >> gpurun_out/r45_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|perm_|gather_agg" >> gpurun_out/r45_kt.txt
done
cat gpurun_out/r45_kt.txt
