#!/bin/bash
# One BASELINE config once per environment setting: TAG=x WL=C2 bash tools/wl_env.sh "A=1" "B=2" ...
O=gpurun_out/${TAG:-wlenv}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
i=0
for setting in "$@"; do
  i=$((i+1))
  echo "$setting" > $O/run_$i.env
  env $setting timeout 900 python bench.py --workload ${WL:-C2} --steps 4 --warmup 3 > $O/run_$i.log 2>&1
done
