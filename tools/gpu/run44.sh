set -x
mkdir -p gpurun_out
export GANN_BATCH_EB=0
GANN_BATCH_DEBUG=1 python tools/ab_search.py --L 128,200 --rounds 1 --reps 5 --var GANN_GTAB_MIN_L=576,64 --var GANN_SEARCH_CARVE=-1,25,40,52,64,77,100 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log; grep "search launch: L" gpurun_out/ab_a.log | sort | uniq -c | sort -k5n | tail -30
