mkdir -p gpurun_out
python tools/diag_timing.py run > gpurun_out/diag_timing.txt 2>&1
rm -f gpurun_out/quick.txt
QUICK_CONFIGS="3" bash tools/gpurun_quick.sh
ncu --set full --import-source on --clock-control none -k regex:"fused_kernel" -c 1 -o gpurun_out/fused_src2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_src2.log 2>&1
