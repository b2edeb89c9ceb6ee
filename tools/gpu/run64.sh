set -x
mkdir -p gpurun_out
GANN_NO_STATS=1 python tools/bench_build.py --reps 2 > gpurun_out/bb_ns.log 2>&1; grep build gpurun_out/bb_ns.log | tail -1
python tools/bench_build.py --reps 2 > gpurun_out/bb_s.log 2>&1; grep build gpurun_out/bb_s.log | tail -1
