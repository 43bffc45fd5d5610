#!/bin/bash
# Profiling recipe (run under gpurun on one B200; see /opt/skills/guides/B200_PROFILING.md).
# 1) plain run of the exact command, 2) ONE ncu invocation: either the launch list
#    (MODE=list) or a full capture of the kernels matching $KERNELS (MODE=full, default).
set -e
CMD="python bench.py --profile --steps 2 --warmup 1"
OUT=${OUT:-gpurun_out}
TAG=${TAG:-prof}
mkdir -p $OUT
$CMD > $OUT/plain.log 2>&1
if [ "${MODE:-full}" = list ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_list.log 2>&1
else
  K=${KERNELS:-k_mlp_bwd_tc|k_encode_fwd|k_encode_bwd}
  N=${COUNT:-$(( $(echo "$K" | tr "|" "\n" | wc -l) + 1 ))}
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s 3 -c $N -o $OUT/$TAG $CMD > $OUT/ncu_$TAG.log 2>&1
fi
