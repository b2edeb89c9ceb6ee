set -x
mkdir -p gpurun_out
for lib in libgann_base.so libgann_b200.so; do
GANN_LIB=$lib python tools/ab_search.py --L 128,200,832 --rounds 2 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|build_ms" gpurun_out/ab_$lib.log
done
ncu --set full --import-source on --clock-control none --profile-from-start off -c 1 -o gpurun_out/search_c1_L832_r02g python tools/ab_search.py --L 832 --profile > gpurun_out/ncu_832.log 2>&1; tail -2 gpurun_out/ncu_832.log
