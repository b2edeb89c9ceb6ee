set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c4_100M_L200 python tools/ab_search.py --config c4 --n 100000000 --L 200 --profile > gpurun_out/ncu_100M.log 2>&1; tail -3 gpurun_out/ncu_100M.log
python tools/ab_search.py --config c4 --n 100000000 --L 200 --rounds 2 > gpurun_out/ab_100M.log 2>&1; grep -E "MQPS|diag|build_ms" gpurun_out/ab_100M.log
python tools/ab_search.py --config c1 --n 10000000 --L 200 --rounds 2 > gpurun_out/ab_10M.log 2>&1; grep -E "MQPS|diag" gpurun_out/ab_10M.log
