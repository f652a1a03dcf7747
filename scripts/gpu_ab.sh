# A/B of an env knob on the attention micro-bench and the in-step sparse timeline.
# usage: KNOB=CSD_PP_WARM VALS="0 1 2" bash scripts/gpu_ab.sh
for v in $VALS; do
  echo "=== $KNOB=$v"
  env $KNOB=$v python scripts/attn_micro.py 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('sparse', r['sparse']['ms'], 'dense', r['dense']['ms'], 'colsum', r['colsum']['ms'])"
  env $KNOB=$v python scripts/step_timeline.py --kind sparse 2>&1 | grep -i "attn\|span\|total" | head -4
done
