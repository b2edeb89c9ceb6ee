set -x
mkdir -p gpurun_out
python tools/ab_search.py --L 128,200 --var GANN_SEARCH_NEXTPF=0,1 --rounds 2 > gpurun_out/ab_200.log 2>&1; grep -E "MQPS|diag|build_ms" gpurun_out/ab_200.log
python tools/ab_search.py --L 832 --var GANN_SEARCH_NEXTPF=0,1 --var GANN_GTAB_LOG2=10,11,12 --rounds 2 > gpurun_out/ab_832.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_832.log
GANN_GTAB_LOG2=11 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -c 1 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_l11.log 2>&1; grep -E "dram__|gpu__time|hit_rate" gpurun_out/ncu_l11.log
python -m pytest tests/test_gpu_baseline.py tests/test_gpu_search.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_s.log 2>&1; tail -2 gpurun_out/t_s.log
