SH="6144x4096,4096x4096,28672x4096,4096x14336"
for diag in 0 1 8 9 32768; do
  TM_PROFILE=1 TM_DIAG=$diag python -m paper_2508_15601_b200.build >/dev/null
  echo "=== TM_DIAG=$diag PDL off"; TM_NO_PDL=1 python scripts/graph_gaps.py 16 $SH 8 | sed -n 2,10p
done
python -m paper_2508_15601_b200.build --force >/dev/null
