# ping-pong attention iteration: parity (bounded), micro-bench, in-step sparse timeline
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_flux_parity.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do timeout 120 python scripts/attn_micro.py 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('sparse', r['sparse']['ms'], 'dense', r['dense']['ms'], 'colsum', r['colsum']['ms'], 'speedup', r['speedup_vs_dense'])"; done
timeout 120 python scripts/step_timeline.py --kind sparse 2>&1 | tail -9
