# Ping-pong attention iteration: attention parity tests, micro-bench of k_attn_pp against
# k_attn_tc (CSD_ATTN_KERNEL=tc), then the per-block timeline of one sparse launch.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "attention or attn or flux" 2>&1 | tail -2
for m in pp tc; do
  r=$(CSD_ATTN_KERNEL=$m timeout 300 python scripts/attn_micro.py 2>&1 | tail -1)
  echo "$m: $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(r["sparse"]["ms"], r["dense"]["ms"], r["speedup_vs_dense"])')"
done
python scripts/attn_pp_trace.py --ctas 1 2>&1 | tee gpurun_out/pp_trace.log
