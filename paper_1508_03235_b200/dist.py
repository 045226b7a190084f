"""Process-group plumbing for row bands across GPUs (DESIGN 8).

One process per GPU (torchrun).  Rank 0 draws an ncclUniqueId from the
library and broadcasts it with torch.distributed; each rank then creates its
band's handle (noc_sim_create with world_size/rank/nccl_id).  The per-cycle
boundary exchange happens inside the library's kernels (CUDA IPC over NVLink);
torch.distributed is only used for this setup and for the bench's timing
reductions.
"""
from __future__ import annotations

import os


def env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def band_rows(mesh_h: int, world: int, rank: int):
    """Rows [row0, row0+rows) of band `rank` of `world`: the library's own
    partition (noc_sim_band_rows; host only)."""
    import ctypes as C
    import paper_1508_03235_b200 as pkg
    a, n = C.c_uint32(), C.c_uint32()
    pkg._check(pkg.lib().noc_sim_band_rows(mesh_h, world, rank, C.byref(a), C.byref(n)))
    return a.value, n.value


def share_nccl_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id() (-> 128 bytes); every rank returns the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def create_band_sim(cfg: dict, device: int, group=None, **kw):
    """Collective: the handle of this rank's band of cfg's mesh."""
    import torch.distributed as dist
    import paper_1508_03235_b200 as pkg
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    nid = share_nccl_id(pkg.noc_sim_nccl_unique_id, group)
    return pkg.NocSim(cfg, device=device, world_size=world, rank=rank, nccl_id=nid, **kw)
