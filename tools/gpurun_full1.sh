# one --set full capture (kept under gpurun's 64 MiB return limit): CFG, KERN regex, TAG
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KERN}" -c ${NK:-2} -f \
  -o gpurun_out/${TAG}_full python bench.py --config ${CFG} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
ls -la gpurun_out/${TAG}_full.ncu-rep
