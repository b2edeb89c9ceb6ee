set -x
mkdir -p gpurun_out
GANN_GTAB_MIN_L=384 ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c1_L832_gtab python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_832g.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c1_L832 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_832.log 2>&1
tail -1 gpurun_out/ncu_832g.log gpurun_out/ncu_832.log
