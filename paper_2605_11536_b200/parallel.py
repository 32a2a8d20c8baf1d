"""Row-band sharding of the frame pipeline over ranks (one process per GPU).

The reference parallelises one frame over image rows with a thread pool
(parallel.hpp:17-36) and its output is bitwise independent of the worker
count (test_pipeline.cpp:80-106).  Here rank g of n owns rows
[g*H/n, (g+1)*H/n); the per-pixel RNG keys stay global (pipeline.hpp:102) so
a band renders exactly what the full frame renders for those rows.  The only
exchange is the spatial-reuse halo: before every spatial pass each rank sends
its `halo` edge rows of the pass-input reservoir grid to its neighbours and
receives theirs (pipeline.hpp:232-269 reads neighbours within
|dy| <= lround(radius) of a snapshot grid).
"""
from __future__ import annotations

import math

import numpy as np


def band_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [y0, y1) owned by `rank` (equal bands, remainder spread from the top)."""
    base, rem = divmod(height, world)
    y0 = rank * base + min(rank, rem)
    return y0, y0 + base + (1 if rank < rem else 0)


def halo_rows(radius: float) -> int:
    """Rows a spatial pass may read beyond a band: neighbor_offset rounds
    rr*sin(th) with rr < radius (pipeline.hpp:232-239), so |dy| <= ceil(radius)."""
    return int(math.ceil(max(0.0, radius)))


def barrier(group) -> None:
    if group is not None:
        import torch.distributed as dist
        dist.barrier(group=group)


def max_over_ranks(x: float, group) -> float:
    if group is None:
        return float(x)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class BandSession:
    """A session rendering one row band of every frame (the whole frame when world == 1)."""

    def __init__(self, renderer, scene_def, cfg, rank: int = 0, world: int = 1, group=None):
        import torch
        if world != 1:
            raise NotImplementedError("row-band sessions for world > 1 are not built yet")
        self.r = renderer
        self.cfg = cfg
        self.rank, self.world, self.group = rank, world, group
        self.sess = renderer.session(scene_def, cfg)
        self.W, self.H = self.sess.width, self.sess.height
        self.y0, self.y1 = band_rows(self.H, world, rank)
        self.stream = torch.cuda.ExternalStream(self.sess.stream_ptr())
        self._pinned = None

    def owned_pixels(self) -> int:
        return (self.y1 - self.y0) * self.W

    def step(self) -> dict:
        return self.sess.step()

    def sync(self) -> None:
        self.sess.sync()

    def timed_steps(self, k: int, stage_tot: list) -> float:
        """Device time (ms) of k frames: CUDA events on the session stream."""
        import torch
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        self.sync()
        start.record(self.stream)
        for _ in range(k):
            self.sess.step()
            _, st = self.sess.last_ms()
            for i in range(6):
                stage_tot[i] += st[i]
        end.record(self.stream)
        end.synchronize()
        return start.elapsed_time(end)

    def read_image_host(self) -> np.ndarray:
        import torch
        if self._pinned is None:
            self._pinned = torch.empty((self.H, self.W, 3), dtype=torch.float64, pin_memory=True).numpy()
        return self.sess.read_image(self._pinned)

    def io_bytes(self):
        return self.sess.io_bytes()

    def halo_launches(self, steps: int) -> int:
        return 0
