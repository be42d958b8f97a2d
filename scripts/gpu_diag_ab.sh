# which stage bounds the decode kernel: disable one at a time (results are wrong; timing only)
for dg in 1 2 4 16 32 3; do
  TM_DIAG=$dg python -m paper_2508_15601_b200.build > /dev/null || { echo "build failed $dg"; continue; }
  echo "== TM_DIAG=$dg"; timeout 120 python scripts/graph_perf.py --ms 16 --mix 2>&1
done
python -m paper_2508_15601_b200.build --force > /dev/null
