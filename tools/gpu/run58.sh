set -x
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/old_c1_L128 python tools/ab_search.py --L 128 --profile > gpurun_out/ncu_o128.log 2>&1; tail -2 gpurun_out/ncu_o128.log
