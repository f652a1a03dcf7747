# tcgen05 GEMM iteration: numerics against torch (pair and single-CTA kernels), block / FLUX
# parity, timings vs cuBLAS, bench line.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_tc.py -q -x 2>&1 | tail -3
CSD_GEMM_PAIR=0 timeout 300 python -m pytest tests/test_gemm_tc.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -k "block or flux or mlp" 2>&1 | tail -2
for m in "CSD_GEMM=tc" "CSD_GEMM_PAIR=0" "CSD_GEMM=cublas"; do env $m timeout 300 python scripts/gemm_micro.py 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/bench.log"):
    if l.startswith("{"):
        r = json.loads(l)
        print("value", r["value"], "dense", r["dense_step_ms"], "sparse", r["sparse_step_ms"], "e2e", r["e2e"]["value"], "attn s/d", r["attention"]["sparse"]["ms"], r["attention"]["dense"]["ms"], "mlp s/d", r["mlp"]["sparse"]["ms"], r["mlp"]["dense"]["ms"])
PY
