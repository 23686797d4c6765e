mkdir -p gpurun_out
TAG=${TAG:-r1c}
CVZ_DEBUG_RESOLVE=1 python scripts/profile_step.py > gpurun_out/resolve_counts_det.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"resolve_coop|relabel_compact|fast_pass|events_coop" -c 4 \
  -o gpurun_out/prof_${TAG} python scripts/profile_step.py --mode fast > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
