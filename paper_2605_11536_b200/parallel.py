"""Row-band sharding of the frame pipeline over ranks (one process per GPU).

The reference parallelises one frame over image rows with a thread pool
(parallel.hpp:17-36) and its output is bitwise independent of the worker
count (test_pipeline.cpp:80-106).  Here rank g of n owns rows
[g*H/n, (g+1)*H/n); the per-pixel RNG keys stay global (pipeline.hpp:102) so
a band renders exactly what the full frame renders for those rows.  The only
exchange is the spatial-reuse halo: before every spatial pass each rank sends
its `halo` edge rows of the pass-input reservoir grid to its neighbours and
receives theirs (pipeline.hpp:232-269 reads neighbours within
|dy| <= lround(radius) of a snapshot grid).  The library packs/unpacks the
rows on its stream (tofr_gpu_session_halo_buffers); the transfer itself is a
torch.distributed batch of isend/irecv (NCCL over NVLink on B200, gloo on
CPU for the tests) enqueued on that same stream.

Temporal reuse reads the previous frame at the reprojected pixel; for a static
camera (every bundled scene) that is the pixel itself, so it stays inside the
band.  For a moving camera the library also exchanges the final grid's halo
(pass -1) and flags any reprojection beyond it as an error.
"""
from __future__ import annotations

import math
import os

import numpy as np


def band_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [y0, y1) owned by `rank` (equal bands, remainder spread from the top)."""
    base, rem = divmod(height, world)
    y0 = rank * base + min(rank, rem)
    return y0, y0 + base + (1 if rank < rem else 0)


def row_weights(image: np.ndarray, shift_cost=None, base: float = 0.05, lit_cost: float = 2.0) -> np.ndarray:
    """Per-row cost of a rendered frame ([H, W, 3]): the shift work counted on
    the device (Newton trials + setup per shift job, by destination row:
    Session.row_cost), the path trees of pixels with a non-zero estimate
    (lit_cost trial-equivalents each) and a little for every pixel (camera
    ray, empty merges)."""
    lit = (np.asarray(image) > 0).any(axis=2).sum(axis=1).astype(np.float64)
    w = lit_cost * lit + base * image.shape[1]
    if shift_cost is not None:
        w = w + np.asarray(shift_cost, dtype=np.float64)
    return w


def balanced_bands(weights, world: int, min_rows: int = 1) -> list:
    """Contiguous row bands [y0, y1) of about equal total weight (cuts at the
    prefix-sum quantiles), each at least max(1, min_rows) rows."""
    w = np.asarray(weights, dtype=np.float64)
    H = len(w)
    m = max(1, int(min_rows))
    if world <= 1:
        return [(0, H)]
    if world * m > H:
        raise ValueError(f"{world} bands of at least {m} rows do not fit {H} rows")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for g in range(1, world):
        y = int(np.searchsorted(cum, cum[-1] * g / world))
        y = max(y, cuts[-1] + m)              # at least m rows in the band above
        y = min(y, H - (world - g) * m)       # room for the bands below
        cuts.append(y)
    cuts.append(H)
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def rebalance_bands(bands, times, min_rows: int = 1) -> list:
    """One refinement step of a row split from measured per-band frame times:
    each band's time is spread evenly over its rows (a piecewise-constant cost
    density), and the rows are cut again at equal cost (balanced_bands)."""
    H = bands[-1][1]
    dens = np.zeros(H)
    for (y0, y1), t in zip(bands, times):
        dens[y0:y1] = float(t) / max(1, y1 - y0)
    return balanced_bands(dens, len(bands), min_rows)


# rows of reprojection margin a band keeps for a moving camera's temporal reuse
# (project() into the previous camera, pipeline.hpp:209-229, may land outside
# the band); a reprojection beyond it raises instead of diverging
MOTION_HALO_ROWS = 16


def halo_rows(radius: float, passes: int = 1, motion_rows: int = 0) -> int:
    """Rows a band keeps on each side: a spatial pass may read |dy| <=
    ceil(radius) rows beyond it (neighbor_offset rounds rr*sin(th) with
    rr < radius, pipeline.hpp:232-239).  Without spatial passes, a moving
    camera's temporal stage still reprojects across band edges: it keeps
    `motion_rows` rows (the spatial halo doubles as that margin otherwise).
    Neither -> no halo."""
    if passes > 0:
        return int(math.ceil(max(0.0, radius)))
    return int(motion_rows)


def motion_rows_for(scene_def, cfg) -> int:
    """MOTION_HALO_ROWS when the camera is animated and temporal reuse is on."""
    cam = getattr(scene_def, "camera", None)
    return MOTION_HALO_ROWS if (cfg.temporal and cam is not None and getattr(cam, "track", None)) else 0


def barrier(group) -> None:
    if group is not None:
        import torch.distributed as dist
        dist.barrier(group=group)


def _dev(group):
    import torch
    import torch.distributed as dist
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"


def max_over_ranks(x: float, group) -> float:
    if group is None:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_floats(xs: list, group) -> list:
    """All ranks' per-frame values (frame latency is the max over the bands
    of the same frame, so the lists are reduced elementwise with MAX)."""
    if group is None:
        return list(xs)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x) for x in xs], dtype=torch.float64, device=_dev(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().tolist()


def gather_floats_all(xs: list, group) -> list:
    """Every rank's values, concatenated in rank order (all_gather)."""
    if group is None:
        return list(xs)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x) for x in xs], dtype=torch.float64, device=_dev(group))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return [float(v) for p in parts for v in p.cpu().tolist()]


class HaloExchanger:
    """Swaps halo rows with the upper (rank-1) and lower (rank+1) neighbour.

    send_lo / recv_lo: this band's first rows / the rows above it (neighbour
    rank-1); send_hi / recv_hi: the band's last rows / the rows below it
    (rank+1).  Tensors are flat byte buffers (device memory owned by the
    library on GPU, plain CPU tensors in the gloo tests)."""

    def __init__(self, rank: int, world: int, group, send_lo, recv_lo, send_hi, recv_hi, stream=None):
        self.rank, self.world, self.group = rank, world, group
        self.send_lo, self.recv_lo, self.send_hi, self.recv_hi = send_lo, recv_lo, send_hi, recv_hi
        self.stream = stream
        self.calls = 0

    def _ops(self):
        import torch.distributed as dist
        ops = []
        if self.rank > 0 and self.send_lo is not None and self.send_lo.numel():
            ops.append(dist.P2POp(dist.isend, self.send_lo, self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self.recv_lo, self.rank - 1, self.group))
        if self.rank < self.world - 1 and self.send_hi is not None and self.send_hi.numel():
            ops.append(dist.P2POp(dist.isend, self.send_hi, self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, self.recv_hi, self.rank + 1, self.group))
        return ops

    def __call__(self, pass_: int = 0) -> None:
        import torch
        import torch.distributed as dist
        ops = self._ops()
        self.calls += 1
        if not ops:
            return
        if self.stream is not None and dist.get_backend(self.group) != "nccl":
            self._host_staged(ops)
        elif self.stream is not None:
            # NCCL waits on the session stream (the pack kernels) and the
            # session stream waits on NCCL (the unpack kernels follow)
            with torch.cuda.stream(self.stream):
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        else:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


    def _host_staged(self, ops) -> None:
        """Device buffers over a host-only backend (gloo): wait for the pack
        kernels, exchange host copies, copy the received rows back."""
        import torch
        import torch.distributed as dist
        self.stream.synchronize()
        host = [op.tensor.cpu() for op in ops]
        for r in dist.batch_isend_irecv([dist.P2POp(op.op, h, op.peer, self.group) for op, h in zip(ops, host)]):
            r.wait()
        with torch.cuda.stream(self.stream):
            for op, h in zip(ops, host):
                if op.op is dist.irecv:
                    op.tensor.copy_(h)


class _DevBytes:
    """__cuda_array_interface__ view of a device allocation owned by the library."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap(ptr: int, nbytes: int, device):
    import torch
    if not ptr or not nbytes:
        return None
    return torch.as_tensor(_DevBytes(ptr, nbytes), device=device)


class BandSession:
    """A session rendering one row band of every frame (the whole frame when world == 1)."""

    def __init__(self, renderer, scene_def, cfg, rank: int = 0, world: int = 1, group=None, plain: bool = False,
                 emulate: bool = False, rows=None, bands=None):
        """emulate: render band `rank` of a `world`-way split alone (no process
        group): the halo exchange is a no-op, so halo rows hold empty
        reservoirs -- the per-GPU work of that split, for one-GPU measurement.
        bands: the split as [(y0, y1)] per rank (default: equal bands,
        band_rows); rows: this rank's band alone (emulation)."""
        import torch
        self.r = renderer
        self.cfg = cfg
        self.plain = plain
        self.rank, self.world, self.group = rank, world, group
        H = scene_def.camera.height
        self.bands = list(bands) if bands else [band_rows(H, world, g) for g in range(world)]
        self.y0, self.y1 = rows if rows else self.bands[rank]
        halo = (halo_rows(cfg.spatial_radius, cfg.spatial_passes, motion_rows_for(scene_def, cfg))
                if (world > 1 and not plain) else 0)
        if world > 1 and min(b[1] - b[0] for b in self.bands) < halo:
            raise ValueError(f"{world} bands of a {H}-row image are thinner than the {halo}-row halo")
        self.halo = halo
        self.sess = renderer.session(scene_def, cfg, band=(self.y0, self.y1, halo), plain=plain)
        self.W, self.H = self.sess.width, self.sess.height
        self.stream = torch.cuda.ExternalStream(self.sess.stream_ptr())
        self.exchanger = None
        if emulate and halo > 0:
            self.sess.set_halo_exchange(lambda pass_: None)
        elif world > 1 and halo > 0 and self._native_nccl(renderer, group):
            pass  # library-side ncclSend / ncclRecv on the session stream, no host callback
        elif world > 1 and halo > 0:
            # host-staged transport (gloo: CPU tests, several ranks sharing one GPU)
            hb = self.sess.halo_buffers()
            dev = torch.device("cuda", torch.cuda.current_device())
            self.exchanger = HaloExchanger(rank, world, group, _wrap(hb["send_lo"], hb["bytes_lo"], dev),
                                           _wrap(hb["recv_lo"], hb["bytes_lo"], dev),
                                           _wrap(hb["send_hi"], hb["bytes_hi"], dev),
                                           _wrap(hb["recv_hi"], hb["bytes_hi"], dev), stream=self.stream)
            self.sess.set_halo_exchange(self.exchanger)
        self._pinned = None

    def _native_nccl(self, renderer, group) -> bool:
        """NCCL process group: hand the library its own communicator (rank 0's
        ncclUniqueId broadcast over the group) so every halo exchange is a
        ncclSend / ncclRecv pair on the session stream.  TOFR_HALO_TRANSPORT=
        callback keeps the torch.distributed callback instead."""
        import torch.distributed as dist
        mode = os.environ.get("TOFR_HALO_TRANSPORT", "native")
        if mode == "callback" or (dist.get_backend(group) != "nccl" and mode != "nccl"):
            return False  # TOFR_HALO_TRANSPORT=nccl: the library's NCCL even on a gloo group
        box = [renderer.nccl_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        if box[0] is None:  # libnccl not loadable by the library: every rank falls back
            return False
        self.sess.halo_nccl(box[0], self.rank, self.world)
        return True

    def halo_transport(self) -> str:
        return self.sess.halo_transport()

    def owned_pixels(self) -> int:
        return (self.y1 - self.y0) * self.W

    def step(self, stats: bool = False):
        return self.sess.step(stats=stats)

    def sync(self) -> None:
        self.sess.sync()

    def timed_steps(self, k: int, stage_tot: list) -> float:
        """Device time (ms) of k frames: CUDA events on the session stream
        around k asynchronous steps; adds the per-stage event sums to stage_tot."""
        import torch
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        self.sync()
        self.sess.stage_totals(reset=True)
        start.record(self.stream)
        for _ in range(k):
            self.sess.step(stats=False)
        end.record(self.stream)
        end.synchronize()
        ms, _, _ = self.sess.stage_totals(reset=True)
        for i in range(6):
            stage_tot[i] += ms[i]
        return start.elapsed_time(end)

    def read_image_host(self) -> np.ndarray:
        """This band's image into pinned host memory (waits for the frame)."""
        import torch
        if self._pinned is None:
            self._pinned = torch.empty((self.y1 - self.y0, self.W, 3), dtype=torch.float64,
                                       pin_memory=True).numpy()
        return self.sess.read_image(self._pinned)

    def run_e2e(self, k: int, warm: int = 0) -> float:
        """k frames through the public API, each frame's image read back to
        pinned host memory (double-buffered: frame f's copy overlaps frame
        f+1's kernels; every copy has landed when this returns).  `warm` frames
        of the same loop run first, untimed.  Steady-state wall seconds of k
        frames, completion to completion: the clock starts when the read-back of
        frame warm-2 lands (frame warm-1 still in flight) and stops when that
        of frame warm+k-2 lands (frame warm+k-1 in flight): k completed frames,
        the pipeline equally full at both ends (timing from the first enqueue
        to the last landing instead counts one to two extra frames of fill and
        drain: -8 to -13% at k = 20, measured)."""
        import time
        import torch
        bufs = [torch.empty((self.y1 - self.y0, self.W, 3), dtype=torch.float64, pin_memory=True).numpy()
                for _ in range(2)]
        self.sync()

        def frame(g):
            self.sess.step(stats=False)
            if g >= 2:
                self.sess.wait_read(g & 1)  # the buffer written two frames ago is free again
            self.sess.read_image_async(bufs[g & 1], g & 1)

        warm = max(warm, 2)
        for g in range(warm):
            frame(g)
        self.sess.wait_read((warm - 2) & 1)  # frame warm-2 landed; warm-1 in flight
        t0 = time.perf_counter()
        for g in range(warm, warm + k):
            frame(g)
        self.sess.wait_read((warm + k - 2) & 1)  # k frames later: warm+k-2 landed
        dt = time.perf_counter() - t0
        self.sess.wait_read((warm + k - 1) & 1)  # drain (untimed)
        self.last_e2e_image = bufs[(warm + k - 1) & 1]
        return dt

    def gather_image(self) -> np.ndarray | None:
        """Full image on rank 0 (None elsewhere): all_gather of the bands."""
        import torch
        import torch.distributed as dist
        band = torch.from_numpy(self.sess.read_image().copy())
        if self.world == 1:
            return band.numpy()
        dev = _dev(self.group)
        hmax = max(b[1] - b[0] for b in self.bands)
        pad = torch.zeros((hmax, self.W, 3), dtype=torch.float64, device=dev)
        pad[: band.shape[0]] = band.to(dev)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        if self.rank != 0:
            return None
        rows = [parts[g][: self.bands[g][1] - self.bands[g][0]] for g in range(self.world)]
        return torch.cat(rows).cpu().numpy()

    def io_bytes(self):
        return self.sess.io_bytes()

    def work(self) -> dict:
        return self.sess.work()

    def halo_launches(self, steps: int) -> int:
        """pack + unpack launches per exchange (one per non-empty side)."""
        if self.exchanger is None:
            return 0
        sides = int(self.rank > 0) + int(self.rank < self.world - 1)
        per_frame = self.cfg.spatial_passes
        return steps * per_frame * 2 * sides
