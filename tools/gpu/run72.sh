set -x
python -m pytest tests/test_gpu_batch.py -m gpu -q -x -p no:cacheprovider -k "tiny" > gpurun_out/t_s.log 2>&1; tail -15 gpurun_out/t_s.log
