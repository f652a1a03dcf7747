# PDL A/B: full GPU suite with PDL on, then attention micro + in-step sparse/dense timelines
# with CSD_PDL=0/1 and CSD_PP_WARM=1/2, and a bench line.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "CSD_PDL=0 CSD_PP_WARM=1" "CSD_PDL=1 CSD_PP_WARM=1" "CSD_PDL=1 CSD_PP_WARM=2"; do
  echo "=== $cfg"
  env $cfg python scripts/attn_micro.py 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('sparse', r['sparse']['ms'], 'dense', r['dense']['ms'], 'colsum', r['colsum']['ms'])"
  env $cfg python scripts/step_timeline.py --kind sparse 2>&1 | tail -10
  env $cfg python scripts/step_timeline.py --kind dense 2>&1 | tail -2
done
CSD_PDL=1 python bench.py --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
