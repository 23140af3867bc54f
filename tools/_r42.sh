./tools/cub_ref 30 > gpurun_out/r42_cub.txt 2>&1
for v in cur pi4 pi16 ct2 ms3 mc4; do
  echo "== $v" >> gpurun_out/r42_kt.txt
  LAPLEX_LIB=$PWD/variants/lib_$v.so timeout 300 python tools/kern_times.py 30 2>&1 | grep -E "total|perm_|main_|sort_count" >> gpurun_out/r42_kt.txt
done
cat gpurun_out/r42_cub.txt gpurun_out/r42_kt.txt
