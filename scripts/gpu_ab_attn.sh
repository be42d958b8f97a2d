# A/B of compile-time variants on the decode attention (scripts/attn_perf.py)
for defs in "$@"; do
  if [ "$defs" = "-" ]; then d=""; else d="$defs"; fi
  TM_DEFS="$d" python -m paper_2508_15601_b200.build --force > /dev/null || { echo "build failed: $d"; continue; }
  echo "== variant [$d]"
  timeout 120 python scripts/attn_perf.py 2>&1 | grep -v "^$"
done
python -m paper_2508_15601_b200.build --force > /dev/null
