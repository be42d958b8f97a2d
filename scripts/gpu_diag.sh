# decode-kernel bottleneck isolation: TM_DIAG bits (1 no W loads, 2 no dequant math, 4 no MMA, 8 no act loads)
for d in 0 1 2 4 8 3 6 9 15; do
  TM_PROFILE=1 TM_DIAG=$d python -m paper_2508_15601_b200.build > /dev/null
  echo "=== TM_DIAG=$d"
  python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "event us|per |   [a-z]"
done
python -m paper_2508_15601_b200.build --force > /dev/null
