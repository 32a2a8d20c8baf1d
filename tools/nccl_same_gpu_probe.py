"""Can the library's NCCL halo transport run two ranks on ONE GPU?  torchrun
--nproc-per-node 2 with a gloo group (several ranks may share cuda:0), the
halo forced through the library's own NCCL communicator
(TOFR_HALO_TRANSPORT=nccl); each rank renders its band and rank 0 compares
the gathered frame with a one-process full-frame render, bit for bit.

    TOFR_HALO_TRANSPORT=nccl torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_same_gpu_probe.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_11536_b200 import _ffi as F  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import GateSpec, RenderConfig, Renderer  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
sd = scenes.bundled("cornell", 48)
cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=2, temporal=True, spatial_passes=2,
                   spatial_neighbors=3, spatial_radius=5, frames=3)
r = Renderer(0)
try:
    bs = parallel.BandSession(r, sd, cfg, rank=rank, world=world, group=dist.group.WORLD)
    print(f"rank {rank}: transport {bs.halo_transport()}", flush=True)
    for _ in range(cfg.frames):
        bs.step()
    bs.sync()
    img = bs.read_image_host().copy()
    parts = [None] * world
    dist.all_gather_object(parts, img)
    if rank == 0:
        got = np.concatenate(parts)
        full = r.session(sd, cfg)
        for _ in range(cfg.frames):
            full.step(stats=False)
        ref = full.read_image()
        print("NCCL_SAME_GPU_OK" if np.array_equal(got, ref) else f"MISMATCH {int((got != ref).sum())}", flush=True)
except Exception as e:  # report, do not hang the other rank
    print(f"rank {rank}: {type(e).__name__}: {e}", flush=True)
dist.destroy_process_group()
