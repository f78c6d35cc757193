"""Debug helper: locate mismatches between the fused path and the oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import depthfill_oracle as O
from paper_1802_00036_b200 import synth, complete_batch
from paper_1802_00036_b200.completion import PipelineConfig, BlurMode, FillMode

cfgs = [("gaussian", "full"), ("none", "full"), ("gaussian", "partial")]
frames = synth.make_batch(1, 100, 8)
for blur, fill in cfgs:
    cfg = PipelineConfig(blur_mode=BlurMode(blur), fill_mode=FillMode(fill))
    res = complete_batch(torch.from_numpy(frames).cuda(), cfg)
    got = res.dense.cpu().numpy()
    for i in range(frames.shape[0]):
        ref, info = O.complete_with_stats(frames[i], O.OracleConfig(blur_mode=O.BlurMode(blur), fill_mode=O.FillMode(fill)), return_stages=True)
        err = np.abs(got[i] - ref)
        bad = np.argwhere(err > 1e-4)
        s5 = info['stages']['extend_top']
        emp = np.argwhere(s5 <= np.float32(0.1))
        print(blur, fill, i, 'max err', err.max(), 'nbad', len(bad), 'iters', int(res.iterations[i]), info['large_fill_iterations'],
              'status', int(res.status[i]), 'empties', len(emp))
        if len(bad):
            ys, xs = bad[:, 0], bad[:, 1]
            print('   bad rows', ys.min(), ys.max(), 'cols', xs.min(), xs.max(), 'first', bad[:8].tolist())
            print('   empties near', [e.tolist() for e in emp[:10]])
