# env A/B on the in-step sparse timeline (3 replays each)
for cfg in $CFGS; do
  echo "=== $cfg"
  env $(echo $cfg | tr ',' ' ') timeout 120 python scripts/step_timeline.py --kind sparse 2>&1 | grep "attn\|k_gemm2_tc<256, true, 1\|span"
done
