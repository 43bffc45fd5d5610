# per-stage device times of the bench step, twice per setting (diagnostic): bash tools/gpu_stages.sh [ENV=... ...]
for cfg in "${@:-DG_X=0}"; do
  for i in 1 2; do env $cfg timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']['stage_ms']; print('$cfg', round(d['ms_per_step'],2), {k: round(v,2) for k,v in r.items()})"; done
done
