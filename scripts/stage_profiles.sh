# Per-kernel stage profiles at C4 (detect, sketch+contract, layout) and one
# ncu --set full capture of the walk.  Usage (under gpurun):
#   TAG=r2c bash scripts/stage_profiles.sh
mkdir -p gpurun_out
TAG=${TAG:-r2}
CFG=${CFG:-C4}
CVZ_DEBUG_RESOLVE=1 timeout 600 python scripts/detect_prof.py $CFG > gpurun_out/detect_${TAG}.log 2>&1
echo "detect rc=$?"
timeout 600 python scripts/contract_prof.py $CFG > gpurun_out/contract_${TAG}.log 2>&1
echo "contract rc=$?"
timeout 600 python scripts/layout_prof.py $CFG 100 > gpurun_out/layout_${TAG}.log 2>&1
echo "layout rc=$?"
if [ -n "$WALK_NCU" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bh_flat_kernel" -s 5 -c 1 \
  -o gpurun_out/walk_${TAG} python scripts/layout_prof.py $CFG 3 > gpurun_out/walk_ncu_${TAG}.log 2>&1
echo "walk ncu rc=$?"
fi
