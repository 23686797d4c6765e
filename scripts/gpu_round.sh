# Bench (N=1, with sharded stages), a 2-rank gloo smoke of the multi-rank bench
# path on one GPU, the ncu launch list and --set full captures of the top
# kernels.  Usage (under gpurun): TAG=r1b bash scripts/gpu_round.sh
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench_${TAG}.log
CVZ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 1 --warmup 3 --config C2 --no-cpu \
  > gpurun_out/bench2_${TAG}.log 2>&1; echo "bench2 rc=$?"; tail -2 gpurun_out/bench2_${TAG}.log
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sharded \
  > gpurun_out/ncu_bench_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"${KREGEX:-bh_flat_kernel|springs_heavy|forces_kernel|update_kernel|slot_counter|relabel_compact|karras}" -c ${KCOUNT:-14} \
  -o gpurun_out/prof_${TAG} python scripts/profile_step.py > gpurun_out/prof_${TAG}.log 2>&1; echo "ncu full rc=$?"
fi
