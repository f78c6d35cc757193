# Quick GPU check (run under gpurun): the GPU test suite, config-1 bench
# lines, QUICK_CONFIGS="0 2 ..." extra configs, and a launch list of config 1.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/quick.txt 2>&1
done
for c in ${QUICK_CONFIGS:-}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/quick.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"r0_kernel|fused_kernel" -c 4 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/quick_ncu.csv 2>&1
