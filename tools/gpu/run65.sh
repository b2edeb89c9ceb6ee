set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python tools/bench_build.py --reps 2 > gpurun_out/bb_s.log 2>&1; grep build gpurun_out/bb_s.log | tail -1
python tools/ab_search.py --L 64,200,832 --rounds 2 --reps 5 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
