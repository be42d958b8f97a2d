for dg in 0 16384; do
  TM_DIAG=$dg python -m paper_2508_15601_b200.build > /dev/null || { echo "build failed $dg"; continue; }
  echo "== TM_DIAG=$dg"; timeout 120 python scripts/graph_perf.py --ms 1,16 --mix 2>&1
done
python -m paper_2508_15601_b200.build --force > /dev/null
