set -x
mkdir -p gpurun_out
for lib in libgann_b200.so libgann_mb8.so; do
GANN_LIB=$lib python tools/bench_build.py --reps 2 > gpurun_out/bb_$lib.log 2>&1; grep -E "build" gpurun_out/bb_$lib.log | tail -1
GANN_LIB=$lib python tools/ab_search.py --L 64,128,200 --rounds 2 --reps 5 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS" gpurun_out/ab_$lib.log
done
