set -x
mkdir -p gpurun_out
for lib in libgann_b200.so libgann_p1.so libgann_p2.so libgann_p3.so; do
GANN_LIB=$lib python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64 --var GANN_BATCH_CARVE=64,77,100 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_$lib.log
done
