# ncu --set full (source-level) of the config-1 fused kernel on 1 %-density frames
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_kernel" -c 1 \
  -o gpurun_out/dens_fused python bench.py --density ${DENS:-0.01} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_dens_fused.log 2>&1
