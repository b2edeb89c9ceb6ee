set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_build.py tests/test_gpu_baseline.py tests/test_gpu_batch.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
GANN_HOST_SHUFFLE=1 python tools/bench_build.py --reps 3 > gpurun_out/bb_host.log 2>&1; grep -E "build" gpurun_out/bb_host.log | tail -4
python tools/bench_build.py --reps 3 > gpurun_out/bb_dev.log 2>&1; grep -E "build" gpurun_out/bb_dev.log | tail -4
