mkdir -p gpurun_out
: > gpurun_out/var.txt
for c in ${CONFIGS:-1 0 2 4}; do
  for v in "" ${VARIANTS}; do
    if [ -z "$v" ]; then lib=paper_1802_00036_b200/libdfc.so; else lib=paper_1802_00036_b200/libdfc_$v.so; fi
    DFC_LIB=$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', '${v:-base}', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/var.txt 2>&1
  done
done
