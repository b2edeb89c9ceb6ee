set -x
for lib in libgann_prev.so libgann_b200.so; do
  GANN_LIB=$lib python tools/bench_build.py --reps 3 > gpurun_out/bb_$lib.log 2>&1; grep -E "build" gpurun_out/bb_$lib.log
done
