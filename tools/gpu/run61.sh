set -x
mkdir -p gpurun_out
export GANN_BATCH_MIN_L=0
python bench.py --points 300000 --queries 4000 --steps 3 --warmup 2 --no-cpu --no-build-roofline > gpurun_out/bench_n1.jsonl 2> gpurun_out/bench_n1.err; echo rc=$?
GANN_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --points 300000 --queries 2000 --steps 3 --warmup 2 --no-cpu --no-build-roofline > gpurun_out/bench_n2.jsonl 2> gpurun_out/bench_n2.err; echo rc=$?; tail -3 gpurun_out/bench_n2.err
GANN_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --points 300000 --queries 2000 --steps 3 --warmup 2 --no-cpu --no-build-roofline --search-on partitions > gpurun_out/bench_n2p.jsonl 2> gpurun_out/bench_n2p.err; echo rc=$?; tail -3 gpurun_out/bench_n2p.err
python - <<'PY'
import json
for f in ('bench_n1','bench_n2','bench_n2p'):
    d=json.loads(open(f'gpurun_out/{f}.jsonl').read().strip().splitlines()[-1])
    print(f, d['n_gpus'], d['value'], d['config'].get('L_search'), d['parity'], d['build'].get('mode'))
PY
