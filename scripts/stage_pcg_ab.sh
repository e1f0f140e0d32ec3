mkdir -p gpurun_out
for rep in 1 2; do for sp in on off; do timeout 300 python scripts/bp5_orders.py --orders 8,9,10,11,12,13,14 --split $sp --out gpurun_out/r2zt_stage_pcg.jsonl > /dev/null 2>&1; done; done
python - <<'PY'
import json
for l in open("gpurun_out/r2zt_stage_pcg.jsonl"):
    d=json.loads(l)
    if "N" in d: print(d["N"], d.get("split"), d["ms_per_iteration"])
PY
