# iteration run: parity tests for the kernels under work + a bench line
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; python - <<'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        r = json.loads(l)
        print({k: r[k] for k in ("value", "dense_step_ms", "sparse_step_ms", "e2e")}, r["attention"]["sparse"]["ms"], r["attention"]["dense"]["ms"], r["attention"]["speedup_vs_dense"])
    else:
        print(l.rstrip()[-300:])
PY
