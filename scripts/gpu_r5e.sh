# community pass + contract ncu --set full capture of the current code
# (session 5); summarised on the box (the report itself exceeds gpurun's
# 64 MiB copy-back)
mkdir -p gpurun_out/prof
timeout 1500 ncu --set full --clock-control none \
  -k regex:"topt|edge_role|events_|resolve_coop|compose|relabel_compact|size_hist|pack_map|compact_edges|degree_hot|cross_keys|add_staged|DeviceRadixSortOnesweep|DeviceReduceByKey" \
  -c 60 -o /tmp/prof_r5e_community python scripts/profile_step.py > gpurun_out/prof_r5e.log 2>&1
echo "ncu full rc=$?"
cp profiles/ncu_traffic.json profiles/ncu_limits.json gpurun_out/prof/ 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof/r5e_ncu_full_c4_community.md /tmp/prof_r5e_community.ncu-rep
echo "summary rc=$?"
