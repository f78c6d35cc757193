# A/B timing of experimental libdfc variants (tools/build_variant.py) on config 1
mkdir -p gpurun_out
for v in "" ${VARIANTS}; do
  if [ -z "$v" ]; then lib=paper_1802_00036_b200/libdfc.so; else lib=paper_1802_00036_b200/libdfc_$v.so; fi
  for rep in 1 2; do
    DFC_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-base}', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/var.txt 2>&1
  done
done
