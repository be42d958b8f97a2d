# A/B of compile-time variants on the decode shapes (CUDA-graph timing):
#   bash scripts/gpu_ab.sh "DEFS_A" "DEFS_B" ...      ("-" = defaults)
mkdir -p gpurun_out
for defs in "$@"; do
  if [ "$defs" = "-" ]; then d=""; else d="$defs"; fi
  TM_DEFS="$d" python -m paper_2508_15601_b200.build --force > /dev/null || { echo "build failed: $d"; continue; }
  echo "== variant [$d]"
  timeout 300 python scripts/graph_perf.py --ms 1,16 --mix 2>&1
done
python -m paper_2508_15601_b200.build --force > /dev/null
