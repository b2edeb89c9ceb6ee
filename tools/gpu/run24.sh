set -x
python tools/ab_search.py --L 640,704,768,832,896,960,1024,1280,1600 --var GANN_GTAB_MIN_L=0,512 --rounds 2 > gpurun_out/ab_go3.log 2>&1; grep -E "MQPS" gpurun_out/ab_go3.log
