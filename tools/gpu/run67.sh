set -x
mkdir -p gpurun_out
for lib in libgann_b200.so libgann_rs45.so libgann_rs46.so libgann_rs28.so; do
GANN_LIB=$lib python tools/bench_build.py --reps 2 > gpurun_out/bb_$lib.log 2>&1; grep -E "build" gpurun_out/bb_$lib.log | tail -1
done
