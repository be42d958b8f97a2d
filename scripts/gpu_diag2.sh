for d in 0 15 2; do
  TM_PROFILE=1 TM_DIAG=$d python -m paper_2508_15601_b200.build > /dev/null
  echo "=== TM_DIAG=$d"
  python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "per |   [a-z]"
done
python -m paper_2508_15601_b200.build --force > /dev/null
