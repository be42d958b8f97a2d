SH="6144x4096,4096x4096,28672x4096,4096x14336"
TM_PROFILE=1 python -m paper_2508_15601_b200.build >/dev/null
echo "=== M=16 PDL off"; TM_NO_PDL=1 timeout 120 python scripts/graph_gaps.py 16 $SH 8
echo "=== M=16 PDL on"; timeout 120 python scripts/graph_gaps.py 16 $SH 8
python -m paper_2508_15601_b200.build --force >/dev/null
