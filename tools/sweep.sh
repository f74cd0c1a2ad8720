#!/bin/bash
# C5 batch sweep (4K context, Conf-KV+INT8) and the other workload lines, under gpurun.
mkdir -p gpurun_out
R=${1:-r01}
for B in 1 2 4 8 16 32 64 128 256; do
  MS=""
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --batch $B $MS > gpurun_out/${R}_sweep_b$B.json 2>>gpurun_out/${R}_sweep.err
done
python - "$R" <<'PY'
import json, sys, glob
R = sys.argv[1]
rows = []
for B in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    try:
        d = json.loads(open(f"gpurun_out/{R}_sweep_b{B}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(B, "failed", e); continue
    rows.append(dict(batch=B, tok_s=d["value"], us_per_step=d["us_per_step"], attn_frac=d["roofline"]["frac"],
                     attn_gbs=d["roofline"]["achieved"], e2e_tok_s=d["e2e"]["value"]))
    print(rows[-1])
json.dump(rows, open(f"gpurun_out/{R}_sweep.json", "w"), indent=1)
PY
