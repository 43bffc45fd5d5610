O=gpurun_out/order_z
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sample_order.py -x -q > $O/t.log 2>&1; echo rc=$? >> $O/t.log
for w in C1 C2; do timeout 900 python bench.py --workload $w --steps 4 --warmup 3 > $O/$w.log 2>&1; done
timeout 300 python bench.py --steps 10 --warmup 3 > $O/C4w1.log 2>&1
