set -x
mkdir -p gpurun_out
GANN_BATCH_DEBUG=1 python tools/ab_search.py --L 832 --rounds 1 --reps 3 --var GANN_BATCH_CM=64,96,128 --var GANN_BATCH_PAD=0,1024 > gpurun_out/ab_batch.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_batch.log; grep "batch launch" gpurun_out/ab_batch.log | sort | uniq -c
