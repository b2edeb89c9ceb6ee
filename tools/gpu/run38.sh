set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_search.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -3 gpurun_out/t_s.log
python tools/ab_search.py --L 200,832 --rounds 2 --var GANN_BATCH_EB=2,4 --var GANN_BATCH_CM=64,96,128 > gpurun_out/ab_batch.log 2>&1; grep -E "MQPS|diag|Error|error|assert" gpurun_out/ab_batch.log
python tools/ab_search.py --L 64,128,400 --rounds 2 --var GANN_BATCH_EB=0,4 --var GANN_BATCH_CM=64 > gpurun_out/ab_batch2.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_batch2.log
