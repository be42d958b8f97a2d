# round-2 profiles: bench launch list, per-shape traffic, decode + prefill full captures, prefill timings
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/plain_dec.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec_r02 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_full_dec.log 2>&1; echo "full dec $?"
python scripts/prof_one.py 8192 28672 4096 3 > gpurun_out/plain_pre.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 2 -c 1 -o gpurun_out/prof_pre_r02 python scripts/prof_one.py 8192 28672 4096 3 > gpurun_out/ncu_full_pre.log 2>&1; echo "full pre $?"
timeout 300 python scripts/prefill_perf.py > gpurun_out/prefill_perf.log 2>&1; echo "pp $?"
