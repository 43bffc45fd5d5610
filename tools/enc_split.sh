#!/bin/bash
# Per-pass encode timings (one launch per pass) under ncu: TAG=x bash tools/enc_split.sh [ENV=VAL ...]
O=gpurun_out/${TAG:-split}; mkdir -p $O
env "$@" DG_ENC_SPLIT_LAUNCH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex_op_red.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_encode -s ${SKIP:-24} -c ${COUNT:-24} --csv --log-file $O/enc_split.csv python bench.py --profile --steps 2 --warmup 1 > $O/ncu.txt 2>&1
python tools/enc_split_summary.py $O/enc_split.csv > $O/summary.txt
