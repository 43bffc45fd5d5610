#!/bin/bash
# Bench once per environment setting (one B200, under gpurun): TAG=x bash tools/ab_env.sh "A=1" "A=2 B=3" ...
O=gpurun_out/${TAG:-abenv}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for setting in "$@"; do
  i=$((i+1))
  echo "$setting" > $O/bench_$i.env
  env $setting timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_$i.log 2>&1
done
