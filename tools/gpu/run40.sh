set -x
mkdir -p gpurun_out
for lib in libgann_b200.so libgann_ld1.so libgann_ld2.so; do
GANN_LIB=$lib python tools/ab_search.py --L 832 --rounds 1 --reps 5 --var GANN_BATCH_CM=64 --var GANN_BATCH_PAD=0,128,256,512,1024 > gpurun_out/ab_$lib.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_$lib.log
done
GANN_BATCH_EB=0 python tools/ab_search.py --L 768,800,832 --rounds 1 --reps 5 > gpurun_out/ab_old.log 2>&1; grep -E "MQPS|Error|error|assert" gpurun_out/ab_old.log
