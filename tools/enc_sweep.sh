#!/bin/bash
# Encode pass-budget sweep (DG_ENC_FWD_MB / DG_ENC_BWD_MB) on the default bench workload.
mkdir -p gpurun_out/sweep
for f in 32 48 64 96 128 192; do
  DG_ENC_FWD_MB=$f DG_ENC_BWD_MB=$f timeout 300 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu --no-cpu-stages --render-steps 1 \
    > gpurun_out/sweep/mb_$f.log 2>&1
  python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
for line in open(f"gpurun_out/sweep/mb_{f}.log"):
    if line.startswith("{"):
        d=json.loads(line); st=d["roofline"]["stage_ms"]
        print(f, "fwd", round(st["encode_fwd"],3), "bwd", round(st["encode_bwd"],3), "total", round(st["total"],3))
PY
done
