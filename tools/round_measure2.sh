# GPU job: bench line, probe-consistent ncu captures of the top kernel, launch list, config 4.
set -x
NCU=ncu
python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -c 4000 gpurun_out/bench.log
# dram traffic vs algorithmic bytes of every cfwd_a launch of one T=512 layer (same run as the probe)
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:cfwd_a \
  --csv --log-file gpurun_out/cfwd_a_T512.csv python tools/ncu_top.py --tokens 512 > gpurun_out/cfwd_a_T512_probe.json 2> gpurun_out/ncu_a.err
tail -2 gpurun_out/cfwd_a_T512_probe.json
# one full capture of a T=2048 cfwd_a launch
$NCU --set full --import-source on --clock-control none -k regex:cfwd_a --launch-skip 3000 -c 1 -o gpurun_out/cfwd_a_full -f \
  python tools/ncu_top.py --tokens 2048 > gpurun_out/cfwd_a_full_probe.json 2> gpurun_out/ncu_b.err
tail -2 gpurun_out/cfwd_a_full_probe.json
# launch list of the bench command itself (times are serialised / cold; shares are what matter)
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_T2048.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu --no-configs --no-dce > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out
# config 4: 12 layers at T=2048 on one GPU
python bench.py --layers 12 --steps 1 --warmup 1 --no-cpu --no-configs --no-dce > gpurun_out/bench_12l.log 2>&1; echo b12_rc=$?
tail -c 2500 gpurun_out/bench_12l.log
