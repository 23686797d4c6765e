# compute-sanitizer over scripts/sanitize_workload.py (C1 + C2 inputs).
# Usage (under gpurun): TAG=r2 bash scripts/sanitize.sh
# racecheck / initcheck at C2 take > 20 min: C1 covers every kernel family,
# C2 adds memcheck + synccheck at a size where the multi-CTA / look-back /
# cooperative paths all engage.
mkdir -p gpurun_out
TAG=${TAG:-r2}
CS="compute-sanitizer --target-processes all --print-limit 50"
run() {
  timeout ${3:-900} $CS --tool $1 python scripts/sanitize_workload.py $2 \
    > gpurun_out/san_${TAG}_$1_$2.log 2>&1
  echo "$1 $2 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${TAG}_$1_$2.log | tail -1)"
}
for tool in memcheck racecheck synccheck initcheck; do run $tool C1; done
for tool in memcheck synccheck; do run $tool C2 1200; done
