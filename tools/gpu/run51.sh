set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 832 --rounds 2 --reps 5 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
GANN_LIB=libgann_u4.so python tools/ab_search.py --L 832 --rounds 2 --reps 5 --var GANN_BATCH_CARVE=64,77,100 > gpurun_out/ab_b.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_b.log
