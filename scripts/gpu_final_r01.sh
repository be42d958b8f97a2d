# round-1 final refresh: full GPU suite, smoke, default bench line (+ reference arm), ncu launch
# list / per-shape traffic / full captures of the decode and the tiled (prefill) kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tests_full.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref $?"; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_r01.csv python scripts/prof_traffic.py > gpurun_out/traffic_order.json 2> gpurun_out/traffic.err; echo "traffic $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:w4a16 -c 300 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec_r01 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_full.log 2>&1; echo "full dec $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 2 -c 1 -o gpurun_out/prof_pre_r01 python scripts/prof_one.py 8192 28672 4096 3 > gpurun_out/ncu_full_pre.log 2>&1; echo "full pre $?"
timeout 300 python scripts/quick_perf.py --ms 2048,4096,8192 > gpurun_out/quick_perf_prefill.log 2>&1; echo "qp $?"
timeout 300 python scripts/graph_perf.py --ms 1,8,16 --mix > gpurun_out/graph_perf.log 2>&1; echo "gp $?"
timeout 300 python scripts/mid_sweep3.py > gpurun_out/mid_sweep.log 2>&1; echo "mid $?"
for t in memcheck synccheck racecheck; do timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1; echo "$t $?"; tail -1 gpurun_out/sanitize_$t.log; done
