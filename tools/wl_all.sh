#!/bin/bash
# Every BASELINE config on one B200 (all partitions on the one GPU): TAG=x bash tools/wl_all.sh
O=gpurun_out/${TAG:-wl}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for w in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --workload $w --steps 4 --warmup 3 > $O/$w.log 2>&1
done
