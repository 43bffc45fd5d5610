#!/bin/bash
# Profiling recipe (run under gpurun on one B200; see /opt/skills/guides/B200_PROFILING.md).
# 1) plain run of the exact command, 2) launch list, 3) full capture of the top kernels.
set -e
CMD="python bench.py --profile --steps 2 --warmup 1"
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
$CMD > $OUT/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
for K in ${KERNELS:-k_mlp_bwd k_encode_fwd k_encode_bwd}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $OUT/prof_$K $CMD > $OUT/ncu_$K.log 2>&1 || echo "ncu $K failed"
done
