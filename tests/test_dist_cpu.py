"""The N>1 host path on CPU: two gloo processes agree on the NCCL unique id
the library draws and on the row-band partition (DESIGN 8)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1508_03235_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1508_03235_b200 as pkg
    nid = pdist.share_nccl_id(pkg.noc_sim_nccl_unique_id)
    # each rank asks the library for its own band
    out[rank] = (nid, pdist.band_rows(208, world, rank))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_ranks_share_nccl_id_and_bands(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ids = {bytes(out[r][0]) for r in range(world)}
    assert len(ids) == 1 and len(next(iter(ids))) == 128 and any(next(iter(ids)))
    rows = [out[r][1] for r in range(world)]
    assert rows[0][0] == 0 and sum(r for _, r in rows) == 208
    assert all(rows[i][0] + rows[i][1] == rows[i + 1][0] for i in range(world - 1))


def test_band_rows_partition():
    """The library's partition (noc_sim_band_rows) is a contiguous cover of
    the rows with band g starting at floor(g*H/P) (DESIGN 8)."""
    for h in (2, 7, 208, 1024):
        for w in range(1, min(h, 8) + 1):
            rows = [pdist.band_rows(h, w, r) for r in range(w)]
            assert [a for a, _ in rows] == [g * h // w for g in range(w)]
            assert sum(r for _, r in rows) == h and min(r for _, r in rows) >= 1
            assert all(rows[i][0] + rows[i][1] == rows[i + 1][0] for i in range(w - 1))
