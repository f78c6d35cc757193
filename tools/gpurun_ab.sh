# A/B of a fused-kernel variant against the baseline path (env var VAR=1 selects the baseline), config 1 (+ QUICK_CONFIGS)
VAR=${VAR:-DFC_NO_R0W}
mkdir -p gpurun_out
rm -f gpurun_out/quick.txt
for rep in 1 2; do
  for v in new base; do
    if [ $v = base ]; then export $VAR=1; else unset $VAR; fi
    for c in 1 ${QUICK_CONFIGS:-}; do
    timeout 120 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c $v', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/quick.txt 2>&1
    done
  done
done
unset $VAR
cat gpurun_out/quick.txt
if [ -n "${WITH_TESTS:-}" ]; then
timeout 600 python -m pytest tests -m gpu -x -q --timeout 180 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
