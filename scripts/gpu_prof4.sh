mkdir -p gpurun_out
TAG=${TAG:-r1d}
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"bh_flat|com_kernel|springs_heavy|add_staged|cross_keys|forces_kernel" -c 8 \
  -o gpurun_out/prof_${TAG} python scripts/profile_step.py > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu rc=$?"
