set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -k "partition or part_batch" > gpurun_out/t_part.log 2>&1; tail -15 gpurun_out/t_part.log
python tools/ab_search.py --L 832,1024 --var GANN_HASH_PER_BEAM=2,4,8,16 --rounds 2 > gpurun_out/ab_hash.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_hash.log
python tools/ab_search.py --L 200 --rounds 2 > gpurun_out/ab_200.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_200.log
