# ncu --set full (source-level) of one config-4 fused-kernel round (PRE + DENSE, 4 strips)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_kernel" -c 1 \
  -o gpurun_out/c4_fused python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4_fused.log 2>&1
