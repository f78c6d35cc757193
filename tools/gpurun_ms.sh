mkdir -p gpurun_out; rm -f gpurun_out/ms.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "multiscale or rounds or config or smoke or baseline" > gpurun_out/pytest_ms.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_ms.log; tail -3 gpurun_out/pytest_ms.log
for rep in 1 2; do
  for c in 2 4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/ms.txt 2>&1
  done
done
cat gpurun_out/ms.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ms_fast|fused_kernel|blur_tail|r0_" -c 8 --csv python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ms_ncu.csv 2>&1
grep -i "ms_fast\|fused\|blur_tail\|r0_" gpurun_out/ms_ncu.csv | awk -F'","' '{print $5, $NF}' | tail -8
