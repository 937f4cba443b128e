# GPU job: nonlinear tests, 2-rank torchrun bench on one GPU (device data plane), config-5 sweep.
set -x
timeout 900 python -m pytest tests/test_gpu_nonlinear.py tests/test_boot.py -m gpu -q -s 2>&1 | tail -12
AEGIS_FORCE_DEVICE=0 AEGIS_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --tokens 512 --steps 1 --warmup 1 --no-dce --no-configs \
  > gpurun_out/bench_2rank.log 2>&1; echo b2_rc=$?
tail -c 2500 gpurun_out/bench_2rank.log
timeout 1200 python tools/sweep.py --out gpurun_out/sweep.txt > gpurun_out/sweep.log 2>&1; echo sweep_rc=$?
cat gpurun_out/sweep.txt
