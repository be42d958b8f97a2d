# current decode breakdown: TM_PROFILE timelines for the 4 shapes at M=16 and M=1, then one ncu --set full
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
( TM_PROFILE=1 python -m paper_2508_15601_b200.build > /dev/null
for shp in "16 28672 4096" "16 4096 4096" "16 6144 4096" "16 4096 14336" "1 4096 4096"; do echo "== $shp"; python scripts/trace_gemm.py $shp 2>&1 | grep -vE "^slowest|^   [0-9]|CTA start ns"; done ) > gpurun_out/trace_r2.log 2>&1
python -m paper_2508_15601_b200.build --force > /dev/null
ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec_r2 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_full.log 2>&1; echo "full $?"
