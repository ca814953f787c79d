"""Multi-rank host logic on CPU (gloo, world size 2 and 4): the block ownership that each rank
derives from the cyclic K_P plan tiles the P x P block-lower-triangular structure exactly once
with balanced work, the distributed product protocol (owned-block partial products +
sum over ranks, the reduce-scatter/all-gather of the GPU path) equals the serial product, and the
NCCL unique id travels through torch.distributed the way bench.py/stbem.Comm bootstrap it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_05224_b200 import stbem as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        P = 2 * world
        own = S.plan_owned_blocks(P, world, rank)
        allown = [None] * world
        dist.all_gather_object(allown, own)
        res["own"] = allown
        # work units on C3 geometry: entries of each owned block (diagonal blocks are triangles)
        first = S.slice_ranges(256, P)
        work = sum(sum(min(a, first[J + 1] - 1) - first[J] + 1 for a in range(first[I], first[I + 1]))
                   for I, J in own)
        allwork = [None] * world
        dist.all_gather_object(allwork, work)
        res["work"] = allwork
        # distributed block-triangular product: partial over owned blocks, then sum over ranks
        ng, nt = 5, 2 * P + 1
        rng = np.random.default_rng(1811)
        A = np.tril(rng.uniform(-1, 1, (nt, nt)))                # block pattern b <= a
        A = np.kron(A != 0, np.ones((ng, ng))) * rng.uniform(-1, 1, (nt * ng, nt * ng))
        x = rng.uniform(-1, 1, nt * ng)
        f = S.slice_ranges(nt, P)
        y = np.zeros(nt * ng)
        for I, J in own:
            r = slice(f[I] * ng, f[I + 1] * ng)
            c = slice(f[J] * ng, f[J + 1] * ng)
            y[r] += A[r, c] @ x[c]
        t = torch.tensor(y)
        dist.all_reduce(t)
        res["matvec_err"] = float(np.abs(t.numpy() - A @ x).max() / np.abs(A @ x).max())
        # NCCL unique id bootstrap (bytes from rank 0, broadcast over the process group)
        uid = [None]
        if rank == 0:
            import ctypes
            buf = ctypes.create_string_buffer(128)
            st = S.lib().bem_nccl_get_unique_id(buf)
            uid = [bytes(buf.raw) if st == S.BEM_OK else b"unavailable"]
        dist.broadcast_object_list(uid, src=0)
        alluid = [None] * world
        dist.all_gather_object(alluid, uid[0])
        res["uid"] = alluid
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_plan_and_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), q), nprocs=world, join=True, start_method="spawn")
    res = q.get(timeout=60)
    P = 2 * world
    blocks = [b for r in res["own"] for b in r]
    assert sorted(blocks) == sorted((i, j) for i in range(P) for j in range(i + 1))   # tiled once
    for r in range(world):                                    # one diagonal block per process p
        assert sum(1 for (i, j) in res["own"][r] if i == j) == P // world
    w = res["work"]
    assert max(w) <= 1.02 * min(w)                           # balanced (P = 2G)
    assert res["matvec_err"] <= 1e-13
    assert len(set(res["uid"])) == 1 and len(res["uid"][0]) in (128, len(b"unavailable"))
