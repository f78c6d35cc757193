"""Sweep HostPipeline chunk size / stream count for the end-to-end (pinned host -> GPU -> pinned host) rate, config 1."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_00036_b200 import synth  # noqa: E402
from paper_1802_00036_b200.completion import BlurMode, FillMode, HostPipeline, PipelineConfig  # noqa: E402

B = 1024
frames = synth.make_batch(1, 0, 16)
host = torch.from_numpy(np.concatenate([frames] * (B // 16))).pin_memory()
out = torch.empty_like(host).pin_memory()
cfg = PipelineConfig(blur_mode=BlurMode.GAUSSIAN, fill_mode=FillMode.FULL)
for chunk in (8, 16, 32, 64, 128):
    for ns in (2, 3, 4, 6):
        pipe = HostPipeline(cfg, chunk=chunk, n_streams=ns)
        for _ in range(2):
            pipe.run(host, out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            pipe.run(host, out)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"chunk {chunk:4d} streams {ns}: {B / dt:9.0f} frames/s  ({2 * host.numel() * 4 / dt / 1e9:.1f} GB/s both ways)", flush=True)
