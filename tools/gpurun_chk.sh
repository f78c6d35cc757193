mkdir -p gpurun_out; rm -f gpurun_out/chk.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
for rep in 1 2; do
  for c in 1 3 0 2 4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'])" >> gpurun_out/chk.txt 2>&1
  done
done
cat gpurun_out/chk.txt
