set -x
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -2 gpurun_out/t_gpu.log
for lib in libgann_prev.so libgann_b200.so; do
  GANN_LIB=$lib python tools/bench_build.py --reps 2 > gpurun_out/bb_$lib.log 2>&1; grep -E "build 1" gpurun_out/bb_$lib.log
  GANN_LIB=$lib python tools/ab_search.py --L 128,200,832 --rounds 2 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS" gpurun_out/ab_$lib.log
done
