# Attention iteration: parity tests for the attention kernels, micro-bench with both staging
# paths (cp.async copy warps vs TMA gather4), then the bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "attention or attn or block or smoke or flux" > gpurun_out/pytest_attn.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_attn.log
for m in cp g4; do
  CSD_ATTN_GATHER=$m timeout 300 python scripts/attn_micro.py > gpurun_out/attn_micro_$m.log 2>&1
  echo "== $m rc=$?"; tail -c 600 gpurun_out/attn_micro_$m.log
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo "bench rc=$?"; python - <<'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        r = json.loads(l)
        print({k: r[k] for k in ("value", "dense_step_ms", "sparse_step_ms")}, r["e2e"]["value"], r["attention"]["sparse"]["ms"], r["attention"]["dense"]["ms"], r["attention"]["speedup_vs_dense"], r["mlp"]["sparse"]["ms"])
    else:
        print(l.rstrip()[-300:])
PY
