mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r5b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gputest_r5b.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r5b.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r5b.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r5b.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_r5b.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r5b.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sharded > gpurun_out/ncu_bench_r5b.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"bh_flat_kernel|springs_heavy|forces_kernel|update_kernel|gather_scan|node_sums|karras|tree_sort|preorder|keys_kernel" -c 24 -o gpurun_out/prof_r5b_layout python scripts/profile_step.py > gpurun_out/prof_r5b.log 2>&1; echo "ncu full rc=$?"
