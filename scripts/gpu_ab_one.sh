# A/B of compile-time variants on one decode shape (CUDA-graph timing):
#   SHAPES=gate_up MS=1 bash scripts/gpu_ab_one.sh "DEFS_A" "DEFS_B" ...      ("-" = defaults)
mkdir -p gpurun_out
for defs in "$@"; do
  if [ "$defs" = "-" ]; then d=""; else d="$defs"; fi
  TM_DEFS="$d" python -m paper_2508_15601_b200.build --force > /dev/null || { echo "build failed: $d"; continue; }
  echo "== variant [$d]"
  timeout 120 python scripts/graph_perf.py --ms ${MS:-1} --shapes ${SHAPES:-gate_up} 2>&1 | grep -v "^$"
done
python -m paper_2508_15601_b200.build --force > /dev/null
