#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (ours + reference), launch list and full ncu capture.
# Usage (under gpurun): TAG=r02_a bash tools/gpu_round.sh
TAG=${TAG:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
if [ -n "$REF" ]; then timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; fi
if [ -z "$SKIP_NCU" ]; then
  OUT=$O MODE=list bash profiles/run_ncu.sh
  OUT=$O TAG=$TAG KERNELS="${KERNELS:-k_mlp_bwd_tc|k_mlp_fwd_tc|k_encode_fwd|k_encode_bwd|k_adam}" bash profiles/run_ncu.sh
fi
