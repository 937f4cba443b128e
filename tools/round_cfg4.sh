# GPU job: config 4 (12 layers, T = 2048, one GPU) + the default bench line.
set -x
timeout 1500 python bench.py --layers 12 --steps 1 --warmup 1 --no-cpu --no-configs --no-dce > gpurun_out/bench_12l.log 2>&1; echo b12_rc=$?
tail -c 1500 gpurun_out/bench_12l.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -c 5000 gpurun_out/bench.log
