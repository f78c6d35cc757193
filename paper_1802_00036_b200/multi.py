"""Multi-GPU completion of one batch.

Frames are independent, so a batch shards by frame index with no collective
on the data path: device i of N takes the contiguous frame range
``sharding.frame_range(i, N, total=B)`` (strong scaling: a fixed batch split
as evenly as possible, BASELINE config 3's 8192 frames over 1/2/4/8 GPUs).
The reference's own model of parallelism is "one pipeline invocation per
thread across a batch of frames" with identical results for any worker count
(reference SPEC.md:357, :594); here a worker is a GPU.

Two ways to run it:

* ``MultiDevicePipeline`` -- one process, one host thread and one
  ``HostPipeline`` (its own CUDA streams and workspaces) per device; host
  scatter (each thread copies its slice of the pinned input) and gather (each
  writes its slice of the pinned output).
* ``python -m paper_1802_00036_b200.multi`` under torchrun -- one process per
  GPU (RANK / LOCAL_RANK / WORLD_SIZE from the environment); every rank
  completes its frame range of a seeded synthetic batch and writes it out.
  The process group (nccl, or gloo with ``--dfc-backend gloo``) only carries the
  untimed barrier; ``--dfc-device`` pins every rank to one GPU, which is how the
  single-GPU test box checks that N ranks reproduce 1 rank bit for bit.
"""

from __future__ import annotations

import argparse
import threading
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .completion import HostPipeline, MultiscaleConfig, PipelineConfig, raise_for_status, _max_depth
from .sharding import env_rank_world, frame_range


class MultiDevicePipeline:
    """Complete [B, H, W] host frames on several devices at once.

    ``devices``: CUDA device indices (default: every visible device).  A
    device may be listed more than once (independent pipelines on one GPU).
    """

    def __init__(self, config: PipelineConfig | None = None, multiscale: MultiscaleConfig | None = None,
                 devices=None, chunk: int = 64, n_streams: int = 3):
        if not torch.cuda.is_available():
            raise RuntimeError("MultiDevicePipeline needs CUDA devices (no CPU fallback)")
        self.config = config or PipelineConfig()
        self.devices = list(range(torch.cuda.device_count())) if devices is None else [int(d) for d in devices]
        if not self.devices:
            raise ValueError("no devices")
        self.pipes = []
        for d in self.devices:
            with torch.cuda.device(d):
                self.pipes.append(HostPipeline(self.config, multiscale, chunk=chunk, n_streams=n_streams, device=d))

    def run(self, host_in: torch.Tensor, host_out: torch.Tensor | None = None, raise_on_error: bool = True):
        """host_in: [B, H, W] float32 CPU tensor (pinned for full overlap).
        Returns (host_out, status[B] int32, iterations[B] int32), all on the CPU."""
        if host_in.dim() == 2:
            host_in = host_in.unsqueeze(0)
        B, H, W = host_in.shape
        if host_out is None:
            host_out = torch.empty((B, H, W), dtype=torch.float32, pin_memory=True)
        status = torch.zeros(B, dtype=torch.int32)
        iters = torch.zeros(B, dtype=torch.int32)
        n = len(self.pipes)
        errors: list[BaseException] = []

        def work(i):
            a, b = frame_range(i, n, total=B)
            if a == b:
                return
            try:
                with torch.cuda.device(self.devices[i]):
                    _, st, it = self.pipes[i].run(host_in[a:b], host_out[a:b], raise_on_error=False)
                status[a:b] = st
                iters[a:b] = it
            except BaseException as e:  # noqa: BLE001
                errors.append(e)

        threads = [threading.Thread(target=work, args=(i,)) for i in range(n)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        if raise_on_error:
            raise_for_status(status.numpy(), _max_depth(self.config))
        return host_out, status, iters


def _main():
    ap = argparse.ArgumentParser(description="frame-sharded completion of a seeded synthetic batch, one rank per GPU "
                                 "(options are --dfc-* so torchrun's own option prefixes never match them)")
    ap.add_argument("--dfc-config", type=int, default=1, help="BASELINE.json config id (synth.CONFIG_SPECS)")
    ap.add_argument("--dfc-first", type=int, default=0, help="first frame index of the batch")
    ap.add_argument("--dfc-total", type=int, required=True, help="frames in the whole batch (split over the ranks)")
    ap.add_argument("--dfc-blur", default="gaussian")
    ap.add_argument("--dfc-fill", default="full")
    ap.add_argument("--dfc-multiscale", action="store_true")
    ap.add_argument("--dfc-out", required=True, help="directory for rank<r>.npz (frames a..b, outputs, status)")
    ap.add_argument("--dfc-device", type=int, default=None, help="pin every rank to this GPU (default LOCAL_RANK)")
    ap.add_argument("--dfc-backend", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()

    import torch.distributed as dist

    from . import synth
    from .completion import BlurMode, FillMode, complete_batch

    rank, local, world = env_rank_world()
    dev = torch.device("cuda", local if args.dfc_device is None else args.dfc_device)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dfc_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    a, b = frame_range(rank, world, total=args.dfc_total)
    frames = synth.make_batch(args.dfc_config, args.dfc_first + a, b - a)
    spec = synth.CONFIG_SPECS[args.dfc_config]
    cfg = PipelineConfig(blur_mode=BlurMode(args.dfc_blur), fill_mode=FillMode(args.dfc_fill), max_depth=float(spec.max_depth))
    res = complete_batch(frames, cfg, multiscale=MultiscaleConfig() if args.dfc_multiscale else None,
                         raise_on_error=False)
    out = Path(args.dfc_out)
    out.mkdir(parents=True, exist_ok=True)
    np.savez(out / f"rank{rank}.npz", start=a, stop=b, dense=res.dense.cpu().numpy(), status=res.status.cpu().numpy(),
             iterations=res.iterations.cpu().numpy(), launches=np.int64(_lib.load().dfc_kernel_launches()))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    _main()
