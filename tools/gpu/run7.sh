set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 832,1024 --var GANN_HASH_LOG2=9,10,11 --rounds 2 > gpurun_out/ab_hlog.log 2>&1; grep -E "MQPS" gpurun_out/ab_hlog.log
python tools/ab_search.py --L 200 --var GANN_HASH_LOG2=10,11 --rounds 2 > gpurun_out/ab_hlog200.log 2>&1; grep -E "MQPS" gpurun_out/ab_hlog200.log
