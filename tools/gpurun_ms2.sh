mkdir -p gpurun_out
python - > gpurun_out/ms2.txt 2>&1 <<'PY'
import os, time, torch
from paper_1802_00036_b200 import complete_batch, synth
from paper_1802_00036_b200.completion import BlurMode, FillMode, PipelineConfig, MultiscaleConfig
cfg = PipelineConfig(blur_mode=BlurMode.MEDIAN_BILATERAL, fill_mode=FillMode.FULL)
for n in (1, 2, 4, 8, 16, 32):
    x = torch.from_numpy(synth.make_batch(2, 0, n)).cuda()
    for rep in range(2):
      for env in ("1", None, "4"):
        if env: os.environ["DFC_MS_NSEG"] = env
        else: os.environ.pop("DFC_MS_NSEG", None)
        for _ in range(5): complete_batch(x, cfg, multiscale=MultiscaleConfig())
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(50): complete_batch(x, cfg, multiscale=MultiscaleConfig())
        torch.cuda.synchronize()
        print(f"fill_in_multiscale batch {n} nseg {env or 'auto'}: {(time.perf_counter()-t0)/50*1e3:.3f} ms per call")
PY
cat gpurun_out/ms2.txt
