"""Multi-rank host logic on CPU (gloo, world_size 2): frame sharding is
disjoint and complete, timings reduce with max-over-ranks, and each rank's
frames are the ones the single-process generator would produce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_00036_b200.sharding import frame_range, max_over_ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import depthfill_oracle as O
        from paper_1802_00036_b200 import synth

        a, b = frame_range(rank, world, total=total)
        spec = synth.SynthSpec(width=96, height=40, beams=12, density=(0.08, 0.12))
        frames = np.stack([synth.make_frame(spec, [3, i]) for i in range(a, b)])
        dense = np.stack([O.complete(f, O.OracleConfig(blur_mode=O.BlurMode.GAUSSIAN)) for f in frames])
        checksum = float(dense.astype(np.float64).sum())
        mx = max_over_ranks([float(rank + 1), checksum])
        gathered = [None] * world
        dist.all_gather_object(gathered, (a, b, checksum))
        out[rank] = (mx, gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 8])
def test_two_rank_sharding(total):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    (mx0, g0), (mx1, g1) = out[0], out[1]
    assert mx0[0] == mx1[0] == 2.0  # max over ranks
    ranges = sorted((a, b) for a, b, _ in g0)
    assert ranges[0][0] == 0 and ranges[-1][1] == total and ranges[0][1] == ranges[1][0]
    # the sharded run reproduces the single-process result frame for frame
    from oracle import depthfill_oracle as O
    from paper_1802_00036_b200 import synth

    spec = synth.SynthSpec(width=96, height=40, beams=12, density=(0.08, 0.12))
    ref = sum(float(O.complete(synth.make_frame(spec, [3, i]),
                               O.OracleConfig(blur_mode=O.BlurMode.GAUSSIAN)).astype(np.float64).sum())
              for i in range(total))
    assert abs(sum(c for _, _, c in g0) - ref) < 1e-6 * abs(ref)


def test_frame_range_weak_and_strong():
    assert frame_range(3, 8, per_rank=1024) == (3072, 4096)
    rs = [frame_range(r, 8, total=8192) for r in range(8)]
    assert rs[0] == (0, 1024) and rs[-1] == (7168, 8192)
    rs = [frame_range(r, 3, total=10) for r in range(3)]
    assert rs == [(0, 4), (4, 7), (7, 10)]
