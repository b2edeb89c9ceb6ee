set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_build.py tests/test_gpu_baseline.py tests/test_gpu_limits.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
GANN_SMALL_U2=0 python tools/bench_build.py --reps 2 > gpurun_out/bb_0.log 2>&1; grep -E "build" gpurun_out/bb_0.log | tail -2
GANN_SMALL_U2=1 python tools/bench_build.py --reps 2 > gpurun_out/bb_1.log 2>&1; grep -E "build" gpurun_out/bb_1.log | tail -2
