set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/gputests.log
for p in imad_peak bfly_peak mix_peak; do timeout 120 tools/probe/$p > gpurun_out/$p.txt 2>&1; cat gpurun_out/$p.txt; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.log
