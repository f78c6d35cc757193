# bench config 1 with each libdfc variant in $VARIANTS (paper_1802_00036_b200/libdfc_NAME.so); "base" = the in-tree lib with $BASE_ENV=1
mkdir -p gpurun_out
rm -f gpurun_out/variants.txt
for rep in 1 2; do
for v in $VARIANTS; do
  if [ $v = base ]; then export ${BASE_ENV:-DFC_NO_R0W}=1; unset DFC_LIB; else unset ${BASE_ENV:-DFC_NO_R0W}; export DFC_LIB=paper_1802_00036_b200/libdfc_$v.so; fi
  timeout 120 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 $v', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/variants.txt 2>&1
done
done
cat gpurun_out/variants.txt
