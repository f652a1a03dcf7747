# CTA-pair attention iteration: parity tests first (bounded), trace, then the micro-bench A/B.
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "prod_sparse_delta" 2>&1 | tail -2
timeout 120 python scripts/attn_cp_trace.py --blocks 14 > gpurun_out/cp_tr.log 2>&1
for v in ${CP_VARIANTS:-"CSD_CP_POLY=0"}; do
  echo "=== $v"
  env $v timeout 120 python scripts/attn_micro.py 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('sparse', r['sparse']['ms'], 'dense', r['dense']['ms'], 'speedup', r['speedup_vs_dense'])"
done
