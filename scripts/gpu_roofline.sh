# Per-kernel roofline metrics of one instrumented pipeline step (every kernel
# name's first launch is tabulated by scripts/roofline_table.py).  Usage
# (under gpurun): TAG=r1k bash scripts/gpu_roofline.sh
mkdir -p gpurun_out
TAG=${TAG:-r1}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
M=$M,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size
timeout 1500 ncu --metrics "$M" --clock-control none -c ${KCOUNT:-600} -o gpurun_out/roof_${TAG} \
  python scripts/profile_step.py > gpurun_out/roof_${TAG}.log 2>&1; echo "ncu roofline rc=$?"
