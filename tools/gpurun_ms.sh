mkdir -p gpurun_out; rm -f gpurun_out/ms.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for c in 2 4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c auto', d['value'], d['roofline']['kernel_ms_per_launch'])" >> gpurun_out/ms.txt 2>&1
  done
done
# single-frame / small-batch latency of fill_in_multiscale (stage 2 segments fill the SMs)
python - >> gpurun_out/ms.txt 2>&1 <<'PY'
import os, time, torch
from paper_1802_00036_b200 import complete_batch, synth
from paper_1802_00036_b200.completion import BlurMode, FillMode, PipelineConfig, MultiscaleConfig
cfg = PipelineConfig(blur_mode=BlurMode.MEDIAN_BILATERAL, fill_mode=FillMode.FULL)
for n in (1, 8):
    x = torch.from_numpy(synth.make_batch(2, 0, n)).cuda()
    for env in ("1", None):
        if env: os.environ["DFC_MS_NSEG"] = env
        else: os.environ.pop("DFC_MS_NSEG", None)
        for _ in range(3): complete_batch(x, cfg, multiscale=MultiscaleConfig())
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20): complete_batch(x, cfg, multiscale=MultiscaleConfig())
        torch.cuda.synchronize()
        print(f"fill_in_multiscale batch {n} nseg {'1' if env else 'auto'}: {(time.perf_counter()-t0)/20*1e3:.3f} ms per call")
PY
cat gpurun_out/ms.txt
