set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 320,400,512,640,832,1024,1280,2048 --rounds 2 --reps 5 --var GANN_BATCH_WPB=4,2 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
