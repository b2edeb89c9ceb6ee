set -x
mkdir -p gpurun_out
GANN_BATCH_DEBUG=1 python tools/ab_search.py --L 320,400,512,640,832,1024 --rounds 1 --reps 4 --var GANN_BATCH_CM=64,96 --var GANN_BATCH_L1KB=2,3,4,6 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
grep "batch launch" gpurun_out/ab_a.log | sort | uniq -c | grep -v "L 128"
