set -x
python tools/ab_search.py --L 832 --var GANN_HASH_LOG2=8,9,10 --rounds 2 > gpurun_out/ab_h.log 2>&1; grep -E "MQPS" gpurun_out/ab_h.log
python tools/ab_search.py --L 640 --var GANN_HASH_LOG2=9,10 --var GANN_GTAB_MIN_L=0,512 --rounds 2 > gpurun_out/ab_h2.log 2>&1; grep -E "MQPS" gpurun_out/ab_h2.log
