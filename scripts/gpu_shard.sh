# Token-sharded block: GPU parity (simulated shards), full GPU suite, the sharded bench path
# at world 1 (torchrun) against the unsharded bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_token_shard.py tests/test_shard.py -q -x 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --sharded --no-cpu-baseline > gpurun_out/bench_token1.log 2>&1; echo "token rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --sharded --shard-mode column --no-cpu-baseline > gpurun_out/bench_col1.log 2>&1; echo "column rc=$?"
for f in bench_token1 bench_col1; do python - $f <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}.log"):
    if l.startswith("{"):
        r = json.loads(l); print(sys.argv[1], r["value"], r["dense_step_ms"], r["sparse_step_ms"], r["config"]["parallelism"])
PY
done
