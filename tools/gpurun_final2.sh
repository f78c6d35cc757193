# Round-2 close measurement set: GPU tests, smoke, every config's bench line
# (config 1 twice: the driver's default command), the reference arm, launch
# lists with DRAM bytes per config, ncu --set full of the config-1 fused kernel
# and the config-0 / config-2 blur tails.
set -x
TAG=${TAG:-r2final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
if [ -z "${NO_TESTS:-}" ]; then
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
fi
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_c1b.log 2>&1
for c in 0 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_c$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.log 2>&1
NO_FULL=${NO_FULL:-} TAG=$TAG bash tools/gpurun_r2_profile.sh
if [ -z "${NO_FULL:-}" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"blur_tail" -c 1 \
  -o gpurun_out/${TAG}_c0_full python bench.py --config 0 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_c0.log 2>&1
fi
