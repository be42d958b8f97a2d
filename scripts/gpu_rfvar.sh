mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v"
  TM_LIB_PATH=scripts/so_var/lib_$v.so timeout 300 python scripts/rf_perf.py --ms 1,16 --no-tmem 2>&1
done > gpurun_out/rfvar.log
