set -x
mkdir -p gpurun_out
python tools/bench_build.py --reps 2 > gpurun_out/bb.log 2>&1; grep -E "build" gpurun_out/bb.log | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_build.csv python tools/bench_build.py --reps 1 > gpurun_out/ncu_bb.log 2>&1
python tools/launch_summary.py gpurun_out/launches_build.csv > gpurun_out/launches_build.txt; head -16 gpurun_out/launches_build.txt
python -m pytest tests/test_gpu_build.py tests/test_gpu_baseline.py tests/test_gpu_limits.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
