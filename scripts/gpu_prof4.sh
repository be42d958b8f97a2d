ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec4 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_dec4.log 2>&1; echo "ncu $?"
