set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf -p no:cacheprovider -x > gpurun_out/t_gpu.log 2>&1; tail -8 gpurun_out/t_gpu.log
python tools/ab_search.py --L 200,832 --var GANN_SEARCH_SPEC=0,1 --rounds 2 > gpurun_out/ab_spec.log 2>&1; grep -E "MQPS|diag|build_ms" gpurun_out/ab_spec.log
