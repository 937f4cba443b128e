nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu --format=csv,noheader -lms 100 > gpurun_out/smi.csv &
SMI=$!
python tools/bench_ops.py --which relin,softrot --reps 10 > gpurun_out/var.log 2>&1
kill $SMI
cat gpurun_out/var.log
python - <<'PY'
import collections
rows=[l.strip().split(', ') for l in open('gpurun_out/smi.csv')]
c=collections.Counter((r[0], r[2]) for r in rows if len(r)>3)
for k,v in sorted(c.items(), key=lambda x:-x[1])[:12]: print(v, k)
PY
