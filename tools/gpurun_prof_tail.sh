mkdir -p gpurun_out
for v in "" ${VARIANTS}; do
  if [ -z "$v" ]; then lib=paper_1802_00036_b200/libdfc.so; n=base; else lib=paper_1802_00036_b200/libdfc_$v.so; n=$v; fi
  DFC_LIB=$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:"blur_tail" -c 1 -o gpurun_out/tail_$n python bench.py --config ${CFG:-0} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tail_$n.log 2>&1
done
