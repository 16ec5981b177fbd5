"""Multi-process (torch.distributed gloo, world_size 2, CPU) coverage of the N>1 host logic:
the shard maps the kernels use (exported host functions of libgf.so) partition the pixels / samples
of a frame exactly, and the per-rank accumulators summed by one all-reduce equal the single-process
frame (the exchange bench.py performs with NCCL on GPUs).  DESIGN.md §9."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_05081_b200 import build as B


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _value(pix, sample):
    """deterministic stand-in for one path estimate (the kernels are GPU-only)."""
    return float(np.sin(0.37 * pix + 1.3 * sample) + 2.0)


def _worker(rank, world, port, W, H, spp, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_05081_b200 import gf
    # tile sharding: every pixel exactly once over the ranks (kind 1)
    cover = torch.zeros(W * H, dtype=torch.int64)
    acc = torch.zeros(W * H * 2, dtype=torch.float64)
    n = gf.shard_paths(W, H, 1, rank, world)
    for p in range(n):
        pix = gf.shard_path_pixel(p, W, H, 1, rank, world)
        if pix < 0:
            continue
        assert gf.shard_pixel_owner(pix % W, pix // W, W, H, world) == rank
        cover[pix] += 1
        for s in range(spp):
            v = _value(pix, s)
            acc[2 * pix] += v
            acc[2 * pix + 1] += v * v
    dist.all_reduce(cover)
    tiles = acc.clone()
    dist.reduce(tiles, dst=0)  # bench.py gathers the disjoint tiles on rank 0
    dist.all_reduce(acc)
    if rank == 0:
        assert torch.equal(tiles, acc)
    # replica check of the BVH hash (bench.replica_check): equal hashes pass, one differing rank fails
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    h = 0xFEDCBA9876543210
    assert bench.replica_check(h, dist, "cpu")
    assert not bench.replica_check(h ^ (rank << 40), dist, "cpu")
    # sample sharding: all pixels, samples s with s mod world == rank (kind 2)
    acc2 = torch.zeros(W * H * 2, dtype=torch.float64)
    n2 = gf.shard_paths(W, H, 2, rank, world)
    for s in range(spp):
        if gf.shard_sample_owner(s, world) != rank:
            continue
        for p in range(n2):
            pix = gf.shard_path_pixel(p, W, H, 2, rank, world)
            if pix < 0:
                continue
            v = _value(pix, s)
            acc2[2 * pix] += v
            acc2[2 * pix + 1] += v * v
    dist.all_reduce(acc2)
    if rank == 0:
        torch.save({"cover": cover, "acc": acc, "acc2": acc2}, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(70, 45), (64, 64)])
def test_two_rank_sharding_and_reduction(tmp_path, W, H):
    B.build()
    out = str(tmp_path / "res.pt")
    spp = 3
    mp.spawn(_worker, args=(2, _free_port(), W, H, spp, out), nprocs=2, join=True)
    res = torch.load(out)
    assert torch.all(res["cover"] == 1), "tile sharding must cover each pixel exactly once"
    ref = torch.zeros(W * H * 2, dtype=torch.float64)
    for pix in range(W * H):
        for s in range(spp):
            v = _value(pix, s)
            ref[2 * pix] += v
            ref[2 * pix + 1] += v * v
    assert torch.allclose(res["acc"], ref, rtol=0, atol=1e-9)
    assert torch.allclose(res["acc2"], ref, rtol=1e-12, atol=1e-9)


def test_single_rank_paths_cover_image():
    B.build()
    from paper_2602_05081_b200 import gf
    W, H = 100, 37
    n = gf.shard_paths(W, H, 0, 0, 1)
    pix = [gf.shard_path_pixel(p, W, H, 0, 0, 1) for p in range(n)]
    pix = [q for q in pix if q >= 0]
    assert sorted(pix) == list(range(W * H))
    # warps are 8x4 pixel blocks: the first 32 paths form one block
    blk = [(q % W, q // W) for q in pix[:32]]
    assert {x for x, _ in blk} == set(range(8)) and {y for _, y in blk} == set(range(4))
