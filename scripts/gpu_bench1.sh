mkdir -p gpurun_out
python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench exit $?"
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
python bench.py --impl reference --steps 50 --warmup 3 > gpurun_out/bench_ref1.json 2>&1; echo "ref exit $?"; cat gpurun_out/bench_ref1.json | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 96 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_bench.log
