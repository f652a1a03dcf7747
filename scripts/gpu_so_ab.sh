# A/B of two builds of the library on one box: _var/libcsd_A.so vs _var/libcsd_B.so
# (copied over the in-tree library in turn; B is left in place).  usage: bash scripts/gpu_so_ab.sh
for r in 1 2; do for v in A B; do
  cp _var/libcsd_$v.so paper_2506_03275_b200/libcsd_b200.so
  echo "=== $v (round $r)"
  timeout 120 python scripts/attn_micro.py 2>&1 | tail -1 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print('sparse', r['sparse']['ms'], 'dense', r['dense']['ms'], 'colsum', r['colsum']['ms'])"
  timeout 120 python scripts/step_timeline.py --kind ${KIND:-dense} 2>&1 | grep "${GREP:-attn\|span}"
done; done
