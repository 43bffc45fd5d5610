mkdir -p gpurun_out/ev
for v in base eval3 eval4; do
  if [ $v = base ]; then L=""; else L="DG_LIB=build/var/lib_$v.so"; fi
  env $L timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu --no-cpu-stages --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['render_rays_per_s'], d['workloads']['C5']['render_rays_per_s'] if d.get('workloads') else None)" >> gpurun_out/ev/ab.txt
done
