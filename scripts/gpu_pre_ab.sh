mkdir -p gpurun_out
for v in base a8 s5 s5a8; do
  echo "== $v"
  TM_LIB_PATH=scripts/so_var/lib_$v.so timeout 300 python scripts/prefill_perf.py --ms 2048,8192 2>&1
done > gpurun_out/pre_ab.log
