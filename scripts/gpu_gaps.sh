TM_PROFILE=1 python -m paper_2508_15601_b200.build >/dev/null
SH="6144x4096,4096x4096,28672x4096,4096x14336"
echo "=== PDL on"; python scripts/graph_gaps.py 16 $SH 8
echo "=== PDL off"; TM_NO_PDL=1 python scripts/graph_gaps.py 16 $SH 8
echo "=== o_proj only, PDL on"; python scripts/graph_gaps.py 16 4096x4096 6
python -m paper_2508_15601_b200.build --force >/dev/null
