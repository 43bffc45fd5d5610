#!/bin/bash
# A/B of an env knob on the whole BASELINE workloads: bash tools/wl_ab.sh OUT ENV=VAL ...
O=gpurun_out/${1:-wl_ab}; shift; mkdir -p $O
for e in "$@"; do
  for w in C1 C5 C4; do
    env $e timeout 600 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$e', '$w', d['config'].get('mode'), round(d['value']), round(d['ms_per_step'],2), round(d.get('render_rays_per_s') or 0))" >> $O/ab.txt 2>&1
  done
done
