# GPU job: the whole -m gpu suite (with per-test durations) + smoke.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo tests_rc=$?
tail -45 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
