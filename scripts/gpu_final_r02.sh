# round-2 refresh: full GPU suite, smoke, bench (+ reference arm), ncu launch list / per-shape
# traffic / full captures (decode, prefill, attention, grouped MoE), prefill raster A/B traffic,
# compute-sanitizer over every kernel variant
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tests_full.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref $?"; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_r02.csv python scripts/prof_traffic.py > gpurun_out/traffic_order.json 2> gpurun_out/traffic.err; echo "traffic $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w4a16_dec -s 4 -c 1 -o gpurun_out/prof_dec_r02 python scripts/prof_one.py 16 28672 4096 6 > gpurun_out/ncu_full.log 2>&1; echo "full dec $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w4a16_gemm -s 2 -c 1 -o gpurun_out/prof_pre_r02 python scripts/prof_one.py 8192 28672 4096 3 > gpurun_out/ncu_full_pre.log 2>&1; echo "full pre $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_dec -s 2 -c 1 -o gpurun_out/prof_attn_r02 python scripts/attn_prof_one.py 32 8192 > gpurun_out/ncu_full_attn.log 2>&1; echo "full attn $?"
for b in 1 0; do TM_PREFILL_BAND=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:w4a16_gemm -s 2 -c 1 --csv --log-file gpurun_out/prefill_band$b.csv python scripts/prof_one.py 8192 28672 4096 3 > /dev/null 2>&1; echo "band $b $?"; done
timeout 300 python scripts/prefill_perf.py > gpurun_out/prefill_perf.log 2>&1; echo "pp $?"
timeout 300 python scripts/graph_perf.py --ms 1,8,16 --mix > gpurun_out/graph_perf.log 2>&1; echo "gp $?"
timeout 300 python scripts/moe_perf.py > gpurun_out/moe_perf.log 2>&1; echo "moe $?"
timeout 300 python scripts/attn_perf.py > gpurun_out/attn_perf.log 2>&1; echo "attn $?"
timeout 600 python scripts/sweep_cfg4.py > gpurun_out/sweep_cfg4.log 2>&1; echo "sweep $?"
for t in memcheck synccheck racecheck; do timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1; echo "$t $?"; tail -1 gpurun_out/sanitize_$t.log; done
