# round-2 re-entry baseline: full GPU suite, smoke, bench, bench launch list, per-shape graph timings
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tests_full.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json | cut -c1-600
timeout 300 python scripts/graph_perf.py --ms 1,8,16 --mix > gpurun_out/graph_perf.log 2>&1; echo "gp $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
