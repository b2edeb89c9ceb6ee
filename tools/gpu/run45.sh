set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=96,128 --var GANN_BATCH_CARVE=77,100 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64 --var GANN_BATCH_CARVE=64 --var GANN_BATCH_POLICY=0,1,2 > gpurun_out/ab_b.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_b.log
GANN_LIB=libgann_eb8.so python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64,96,128 --var GANN_BATCH_CARVE=64,77 > gpurun_out/ab_c.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_c.log
