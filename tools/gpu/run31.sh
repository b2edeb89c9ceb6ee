set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c1.jsonl 2> gpurun_out/bench_c1.err; tail -3 gpurun_out/bench_c1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_build_c1.csv python tools/bench_build.py --reps 1 > gpurun_out/ncu_build.log 2>&1; tail -2 gpurun_out/ncu_build.log
