set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_build.py tests/test_gpu_baseline.py tests/test_gpu_limits.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
for i in 1 2 3; do python tools/bench_build.py --reps 1 2>&1 | grep -E "^build" | tail -1; done
