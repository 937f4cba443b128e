# GPU job: the whole -m gpu suite, smoke, per-op profile of the layer, the default bench line.
set -x
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests_rc=$?
tail -25 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke.log
timeout 900 python tools/profile_layer.py --tokens 2048 --out gpurun_out/layer_ops.txt > gpurun_out/layer_ops.log 2>&1; echo prof_rc=$?
head -40 gpurun_out/layer_ops.txt
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -c 1500 gpurun_out/bench.log
