set -x
python tools/ab_search.py --L 640,832,1024 --var GANN_GTAB_ONLY=0,1 --var GANN_GTAB_MIN_L=384 --rounds 2 > gpurun_out/ab_go.log 2>&1; grep -E "MQPS" gpurun_out/ab_go.log
python tools/ab_search.py --L 400,512 --var GANN_GTAB_ONLY=1 --var GANN_GTAB_MIN_L=0,384 --rounds 2 > gpurun_out/ab_go2.log 2>&1; grep -E "MQPS" gpurun_out/ab_go2.log
