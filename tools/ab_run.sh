# GPU job: alternate A/B timing of libaegis variants on the layer's op groups.
#   bash tools/ab_run.sh "<variant names, '' = default build>" [rounds] [which]
# e.g. bash tools/ab_run.sh "default fin0" 3
set -x
vars=${1:-default}; rounds=${2:-3}; which=${3:-rot,relin,softrot}
for r in $(seq 1 $rounds); do
  for v in $vars; do
    if [ "$v" = default ]; then lib=""; else lib=paper_2604_03425_b200/libaegis_$v.so; fi
    echo "== round $r variant $v"
    AEGIS_LIB=$lib timeout 600 python tools/bench_ops.py --which $which --reps 3 2>&1 | grep -v "^ "
  done
done
