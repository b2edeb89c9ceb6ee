set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64,128 --var GANN_BATCH_PAD=0,1024 > gpurun_out/ab_a.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_a.log
python tools/ab_search.py --L 128,200,400 --rounds 1 --reps 5 --var GANN_BATCH_EB=0,4 --var GANN_BATCH_CM=64 > gpurun_out/ab_b.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_b.log
GANN_BATCH_CM=64 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/batch_c1_L832 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_b832.log 2>&1; tail -2 gpurun_out/ncu_b832.log
