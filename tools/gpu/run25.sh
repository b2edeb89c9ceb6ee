set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
python tools/ab_search.py --L 200,832 --rounds 2 > gpurun_out/ab_base.log 2>&1; grep -E "MQPS|diag|build_ms" gpurun_out/ab_base.log
