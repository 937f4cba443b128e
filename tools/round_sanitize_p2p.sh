# GPU job: compute-sanitizer memcheck / racecheck over the device-synchronised PCMM exchange
# (2 processes on one GPU, FFN graph at N = 2^11, T = 16: one token group split over both ranks).
set -x
for t in memcheck racecheck; do
  P2P_TOKENS=16 P2P_KIND=1 P2P_MODE=device timeout 1500 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 2961$([ $t = memcheck ] && echo 1 || echo 2) --no-python \
    compute-sanitizer --tool $t --print-limit 20 python tests/_p2p_worker.py > gpurun_out/sanitize_p2p_$t.txt 2>&1
  echo ${t}_rc=$?
  grep -E "P2P_|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_p2p_$t.txt
done
