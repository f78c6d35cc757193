# quick: selected GPU tests (PYTEST_K) + config-1 bench x2 (+ QUICK_CONFIGS)
mkdir -p gpurun_out
if [ -n "${PYTEST_K:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_quick.log 2>&1; echo "rc $?" >> gpurun_out/pytest_quick.log
fi
: > gpurun_out/quick.txt
for rep in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['roofline']['kernel_ms_per_launch'], d['gpu_launches'])" >> gpurun_out/quick.txt 2>&1
done
for c in ${QUICK_CONFIGS:-}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/quick.txt 2>&1
done
