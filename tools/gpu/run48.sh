set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/batch_c1_L832 python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_b832.log 2>&1; tail -2 gpurun_out/ncu_b832.log
