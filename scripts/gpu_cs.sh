# Dense / column-sum attention kernels: parity tests, then FLUX timings per kernel family
# (default: k_attn_sd for dense passes; CSD_ATTN_DENSE=pp|tc for the others).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "attention or attn or flux or block or colsum" 2>&1 | tail -3
for m in sd pp tc; do
  r=$(CSD_ATTN_DENSE=$m timeout 300 python scripts/attn_micro.py 2>&1 | tail -1)
  echo "$m: $(echo $r | python -c 'import json,sys; r=json.loads(sys.stdin.read()); print(r["sparse"]["ms"], r["dense"]["ms"], r["colsum"], r["speedup_vs_dense"])' 2>&1 | tail -1)"
done
