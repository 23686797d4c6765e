# One GPU sanity pass: parity tests, smoke, a short bench, and the ncu launch list.
# usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [bench-args]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -20 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -20 gpurun_out/bench.log
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
fi
