"""Reference CPU path timed on the host cores -- BASELINE INFRASTRUCTURE ONLY.

Runs the reference algorithm (oracle pipeline orchestration over the
reference's compiled ``_native_ops`` from oracle/_ref when available --
kind "reference" -- else the numpy oracle port -- kind "port") one frame per
task on ``procs`` single-threaded worker processes, as SURVEY.md 8(d)
prescribes.  Used only by bench.py's cpu_baseline leg and ``--impl reference``.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

_FRAMES = None
_CFG = None
_OPS = None


def _init(frames, cfg, kind):
    global _FRAMES, _CFG, _OPS
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import depthfill_oracle as O

    _FRAMES, _CFG = frames, cfg
    if kind == "reference":
        from oracle.ref_ops import RefNativeOps

        _OPS = RefNativeOps
    else:
        _OPS = O.NumpyOps


def _work(i):
    from oracle import depthfill_oracle as O

    O.complete(_FRAMES[i % len(_FRAMES)], _CFG, _OPS)
    return i


def available_kind() -> str:
    try:
        from oracle.ref_ops import load_native

        return "reference" if load_native() is not None else "port"
    except Exception:  # noqa: BLE001
        return "port"


def time_cpu(frames: np.ndarray, cfg, n_frames: int, procs: int | None = None, kind: str | None = None,
             pool=None) -> dict:
    """Complete ``n_frames`` (cycling over ``frames``) on ``procs`` processes.

    Returns {"value": frames/s, "seconds", "frames", "cores", "kind"}."""
    kind = kind or available_kind()
    procs = procs or os.cpu_count() or 1
    own = pool is None
    if own:
        ctx = mp.get_context("fork")
        pool = ctx.Pool(procs, initializer=_init, initargs=(frames, cfg, kind))
    try:
        pool.map(_work, range(procs), chunksize=1)  # warm every worker
        t0 = time.perf_counter()
        pool.map(_work, range(n_frames), chunksize=1)
        dt = time.perf_counter() - t0
    finally:
        if own:
            pool.close()
            pool.join()
    return {"value": n_frames / dt, "seconds": dt, "frames": n_frames, "cores": procs, "kind": kind}


def make_pool(frames, cfg, procs=None, kind=None):
    kind = kind or available_kind()
    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("fork")
    return ctx.Pool(procs, initializer=_init, initargs=(frames, cfg, kind)), procs, kind


def single_frame_seconds(frame, cfg, kind=None) -> float:
    kind = kind or available_kind()
    _init(frame[None], cfg, kind)
    _work(0)
    t0 = time.perf_counter()
    _work(0)
    return time.perf_counter() - t0
