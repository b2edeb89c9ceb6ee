set -x
mkdir -p gpurun_out
GANN_BATCH_DEBUG=1 python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64 --var GANN_BATCH_CARVE=25,40,52,64,77,100 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log; grep "batch launch: L 832" gpurun_out/ab_a.log | sort | uniq -c
