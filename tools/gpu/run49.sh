set -x
mkdir -p gpurun_out
for lib in libgann_b200.so libgann_mb5.so libgann_mb4.so libgann_rb8.so; do
GANN_LIB=$lib python tools/ab_search.py --L 512,832,1280 --rounds 2 --reps 5 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_$lib.log
done
