mkdir -p gpurun_out
TAG=${TAG:-r1b}
CVZ_DEBUG_RESOLVE=1 python scripts/profile_step.py > gpurun_out/resolve_counts_det.log 2>&1
CVZ_DEBUG_RESOLVE=1 python scripts/profile_step.py --mode fast > gpurun_out/resolve_counts_fast.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"resolve_coop|relabel_compact|slot_keys|events_coop|fast_pass" -c 8 \
  -o gpurun_out/prof_${TAG}_det python scripts/profile_step.py --mode fast > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
