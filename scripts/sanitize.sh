# compute-sanitizer over scripts/sanitize_workload.py (C1 + C2 inputs).
# Usage (under gpurun): TAG=r2 bash scripts/sanitize.sh
mkdir -p gpurun_out
TAG=${TAG:-r2}
CS="compute-sanitizer --target-processes all --print-limit 50"
for cfg in C1 C2; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 $CS --tool $tool python scripts/sanitize_workload.py $cfg \
      > gpurun_out/san_${TAG}_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${TAG}_${tool}_${cfg}.log | tail -1)"
  done
done
