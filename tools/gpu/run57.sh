set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 400,832,1280 --rounds 2 --reps 5 --var GANN_GTAB_LOG2=10,11,12 --var GANN_GTAB_KEEP=0,1 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
