set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 200,512,832 --var GANN_SEARCH_SPEC=0,1 --rounds 2 > gpurun_out/ab_spec2.log 2>&1; grep -E "MQPS|build_ms" gpurun_out/ab_spec2.log
