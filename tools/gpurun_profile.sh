# per-warp timing build + one ncu --set full source-level capture of the fused kernel (config 1)
mkdir -p gpurun_out
python tools/diag_timing.py run > gpurun_out/diag_timing.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fused_kernel" -c 1 -o gpurun_out/fused_src3 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_src3.log 2>&1
