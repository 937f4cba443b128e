# GPU job: ncu launch list of the bench command itself (no warm-up, one timed layer, T = 2048).
# Per-launch times are serialised (ncu) and L2 is not flushed: use the kernels' SHARES of the step.
set -x
timeout 3300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
  --log-file gpurun_out/launches_bench_T2048.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu --no-configs --no-dce --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
echo ncu_rc=$?
ls -la gpurun_out/launches_bench_T2048.csv
python tools/kernel_split.py gpurun_out/launches_bench_T2048.csv 1 | head -30
