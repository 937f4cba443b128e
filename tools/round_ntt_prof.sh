# GPU job: NTT v2 timing + one ncu --set full capture of fwd_a / fwd_b / inv_b / inv_a (source-level).
set -x
python tools/bench_ntt.py --shapes 48x17 --impls 1 > gpurun_out/ntt_bench.txt 2>&1; cat gpurun_out/ntt_bench.txt
ncu --set full --import-source on --clock-control none -k "regex:fwd_a|fwd_b|inv_a|inv_b" --launch-skip 8 -c 4 -o gpurun_out/ntt_full -f \
  python tools/bench_ntt.py --shapes 48x17 --impls 1 > gpurun_out/ntt_ncu.log 2>&1
ls -la gpurun_out/ntt_full.ncu-rep
