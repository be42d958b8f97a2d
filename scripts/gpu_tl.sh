TM_PROFILE=1 python -m paper_2508_15601_b200.build > /dev/null
for shp in "16 28672 4096" "16 4096 4096" "16 4096 14336"; do echo "== $shp"; python scripts/trace_gemm.py $shp 2>&1 | grep -E "per |timeline|   |event"; done
