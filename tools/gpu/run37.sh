set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_search.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
python tools/ab_search.py --L 200,832 --rounds 2 --var GANN_BATCH_EB=0,2,4 --var GANN_BATCH_POLICY=1,2 > gpurun_out/ab_batch.log 2>&1; grep -E "MQPS|diag|Error|error|assert" gpurun_out/ab_batch.log
python tools/ab_search.py --L 832 --rounds 2 --var GANN_BATCH_CM=64,128 > gpurun_out/ab_batch2.log 2>&1; grep -E "MQPS|diag|Error|error|assert" gpurun_out/ab_batch2.log
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/batch_c1_L832 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_b832.log 2>&1; tail -2 gpurun_out/ncu_b832.log
