mkdir -p gpurun_out
timeout 600 python scripts/e2_vs_bf16.py > gpurun_out/e2.md 2>&1; echo "e2 $?"; cat gpurun_out/e2.md
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:w4k -c 300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
