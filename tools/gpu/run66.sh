set -x
mkdir -p gpurun_out
GANN_SMALL_U2=0 python tools/bench_build.py --reps 2 > gpurun_out/bb_0.log 2>&1; grep -E "build" gpurun_out/bb_0.log | tail -1
GANN_SMALL_U2=1 python tools/bench_build.py --reps 2 > gpurun_out/bb_1.log 2>&1; grep -E "build" gpurun_out/bb_1.log | tail -1
