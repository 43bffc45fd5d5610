# A/B of library builds / env knobs on the bench's stage times (diagnostic)
run() { env "$@" timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e --no-extra 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']['stage_ms']; print('$*', round(d['ms_per_step'],2), {k: round(v,3) for k,v in r.items() if k in ('segment','march','encode_fwd','mlp_fwd','composite','merge_bwd','encode_bwd','mlp_bwd','adam')})"; }
for cfg in "$@"; do run $cfg; done
