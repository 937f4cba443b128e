# GPU job: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_smoke.py.
set -x
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/sanitize_$t.txt 2>&1
  echo ${t}_rc=$?
  tail -4 gpurun_out/sanitize_$t.txt
done
