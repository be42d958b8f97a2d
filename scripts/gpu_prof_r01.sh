mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_r01.csv python scripts/prof_traffic.py > gpurun_out/traffic_order.json 2> gpurun_out/traffic.err; echo "traffic $?"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:w4a16 -c 300 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec_r01 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_full.log 2>&1; echo "full $?"
