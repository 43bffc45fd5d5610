#!/bin/bash
# Forward grouping of hashed-level passes (DG_ENC_FWD_HGROUP_MB) on C1, C2 and the C4 weak point
O=gpurun_out/${TAG:-grp}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sample_order.py tests/test_gpu_full_size.py -x -q > $O/t.log 2>&1; echo rc=$? >> $O/t.log
for g in ${GS:-64 0}; do
  env "${KNOB:-DG_ENC_FWD_HGROUP_MB}=$g" timeout 900 python bench.py --workload C2 --steps 4 --warmup 3 > $O/C2_$g.log 2>&1
  env "${KNOB:-DG_ENC_FWD_HGROUP_MB}=$g" timeout 300 python bench.py --steps 10 --warmup 3 > $O/C4w1_$g.log 2>&1
  env "${KNOB:-DG_ENC_FWD_HGROUP_MB}=$g" timeout 900 python bench.py --workload C1 --steps 4 --warmup 3 > $O/C1_$g.log 2>&1
done
