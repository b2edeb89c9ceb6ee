set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_batch.py tests/test_gpu_baseline.py tests/test_gpu_checked.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
for lib in libgann_prev.so libgann_b200.so; do
GANN_LIB=$lib python tools/ab_search.py --L 400,832,1280 --rounds 2 --reps 5 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_$lib.log
done
