# ncu captures of the top kernels of one bench step (1 GPU).  Output under gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"bh_kernel|forces_kernel|update_kernel|slot_counter_kernel|relabel_compact|com_kernel" -c 10 \
  -o gpurun_out/prof_${TAG}_det python scripts/profile_step.py > gpurun_out/prof_${TAG}_det.log 2>&1; echo "ncu det rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"fast_pass_kernel" -c 2 \
  -o gpurun_out/prof_${TAG}_fast python scripts/profile_step.py --mode fast > gpurun_out/prof_${TAG}_fast.log 2>&1; echo "ncu fast rc=$?"
tail -3 gpurun_out/prof_${TAG}_det.log gpurun_out/prof_${TAG}_fast.log
