# Round-2 measurement set: every config's ncu launch list (time + DRAM bytes per
# launch; traffic.json comes from these), one --set full capture of the config-1
# fused kernel (source-level) and of the config-2 blur tail, SASS histogram.
# Usage: TAG=r2a bash tools/gpurun_r2_profile.sh
TAG=${TAG:-r2}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${CONFIGS:-1 0 2 3 4}; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}_c$c.log 2>&1
done
if [ -z "${NO_FULL:-}" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_kernel|r0_kernel" -c 2 \
  -o gpurun_out/${TAG}_c1_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur_tail|ms_fast" -c 2 \
  -o gpurun_out/${TAG}_c2_full python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c2.log 2>&1
fi
