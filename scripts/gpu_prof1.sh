mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 4 -c 1 -o gpurun_out/prof_dec_gateup python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_dec.log 2>&1; echo "ncu dec $?"
ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 2 -c 1 -o gpurun_out/prof_pre_gateup python scripts/prof_one.py 8192 28672 4096 3 > gpurun_out/ncu_pre.log 2>&1; echo "ncu pre $?"
ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 4 -c 1 -o gpurun_out/prof_dec_o python scripts/prof_one.py 16 4096 4096 6 > gpurun_out/ncu_dec_o.log 2>&1; echo "ncu dec o $?"
tail -3 gpurun_out/ncu_dec.log
ls -la gpurun_out
