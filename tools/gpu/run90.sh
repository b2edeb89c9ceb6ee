set -x
python tools/ab_search.py --nq 4000 --L 1024,1600,2048,4096,8192 --rounds 1 --reps 2 --var GANN_GTAB_LOG2=11,12 2>&1 | grep -E "MQPS|assert|Error|error"
