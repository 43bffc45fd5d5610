#!/bin/bash
# A/B of the paired ReLU MLP backward against the serial one (DG_MLP_BWD_SERIAL=1), with the
# parity suites that exercise the backward first.  Usage (under gpurun): TAG=pair2 bash tools/ab_pair.sh
O=gpurun_out/${TAG:-pair}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_sample_parity.py} -x -q > $O/t1.log 2>&1; echo rc=$? >> $O/t1.log
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_pair.log 2>&1; echo rc=$? >> $O/bench_pair.log
[ -n "$NO_SERIAL" ] || { DG_MLP_BWD_SERIAL=1 timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_serial.log 2>&1; echo rc=$? >> $O/bench_serial.log; }
