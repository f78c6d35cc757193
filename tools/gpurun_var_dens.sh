mkdir -p gpurun_out
: > gpurun_out/var.txt
for d in "" 0.01; do
  for v in "" ${VARIANTS}; do
    if [ -z "$v" ]; then lib=paper_1802_00036_b200/libdfc.so; else lib=paper_1802_00036_b200/libdfc_$v.so; fi
    for rep in 1 2; do
    DFC_LIB=$lib timeout 300 python bench.py ${d:+--density $d} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('d${d:-def}', '${v:-base}', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/var.txt 2>&1
    done
  done
done
