set -x
python tools/ab_search.py --nq 2000 --L 2048,4096,8192,16384 --rounds 1 --reps 1 --var GANN_BATCH_EB=0,4 2>&1 | grep -E "MQPS|assert|Error|error"
