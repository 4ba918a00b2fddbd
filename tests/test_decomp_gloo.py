"""CPU, world_size 2 (gloo): the host-side logic of the multi-GPU path.

Each rank owns one z-slab laid out exactly like the device Q buffer
([nzl+8 planes][5][n][n]); the ghost planes are exchanged with
torch.distributed send/recv using the byte offsets of mpfd_b200_halo_plan --
the same plan the NCCL path uses (solver.cu halo_refresh).  Checks:
  * ghosts equal the periodic wrap of the global field (fill_halos_periodic's
    z pass, field.cpp:29-36);
  * the rank-ordered gather of 4096-chunk sums followed by the host pairwise
    tree equals the reference's deterministic_sum over the whole field
    (reduce.cpp:24-36), i.e. diagnostics are decomposition independent.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, result_dir):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2505_20911_b200 as m
    import pyoracle as po

    L = m.lib()
    bq = 8
    plan = (C.c_longlong * 9)()
    assert L.mpfd_b200_halo_plan(n, world, rank, bq, plan) == 0
    send_up, recv_lo, send_dn, recv_hi, blk, up, dn, z0, nzl = [int(x) for x in plan]
    rng = np.random.default_rng(7)
    glob = rng.standard_normal((n, 5, n, n))  # [z][comp][y][x]
    q = np.zeros((nzl + 8, 5, n, n))
    q[4:4 + nzl] = glob[z0:z0 + nzl]
    buf = torch.from_numpy(q.reshape(-1).view(np.uint8))
    el = lambda off: off  # byte offsets
    reqs = [
        dist.isend(buf[el(send_up):el(send_up) + blk].clone(), up),
        dist.isend(buf[el(send_dn):el(send_dn) + blk].clone(), dn),
    ]
    lo = torch.empty(blk, dtype=torch.uint8)
    hi = torch.empty(blk, dtype=torch.uint8)
    dist.recv(lo, dn)
    dist.recv(hi, up)
    for r in reqs:
        r.wait()
    buf[recv_lo:recv_lo + blk] = lo
    buf[recv_hi:recv_hi + blk] = hi
    q = buf.numpy().view(np.float64).reshape(nzl + 8, 5, n, n)
    for g in range(4):
        assert np.array_equal(q[g], glob[(z0 - 4 + g) % n])
        assert np.array_equal(q[nzl + 4 + g], glob[(z0 + nzl + g) % n])
    # diagnostics: chunk sums in global scan order, gathered by rank
    Lo = po.oracle_lib()
    integ = np.ascontiguousarray(glob[z0:z0 + nzl, 0]).reshape(-1)
    nch = integ.size // 4096
    parts = np.array([Lo.orc_pairwise_sum(integ[i * 4096:].ctypes.data_as(C.POINTER(C.c_double)), 4096)
                      for i in range(nch)])
    allp = [torch.zeros(nch, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allp, torch.from_numpy(parts))
    allp = torch.cat(allp).numpy()
    got = Lo.orc_pairwise_sum(allp.ctypes.data_as(C.POINTER(C.c_double)), allp.size)
    full = np.ascontiguousarray(glob[:, 0]).reshape(-1)
    want = Lo.orc_deterministic_sum(full.ctypes.data_as(C.POINTER(C.c_double)), full.size, 8)
    assert got == want
    with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_halo_and_reduction(tmp_path, world):
    import paper_2505_20911_b200 as m

    m.lib()  # fail here, not in the workers, if the library is missing
    mp.spawn(_worker, args=(world, _free_port(), 64, str(tmp_path)), nprocs=world, join=True)
    assert all(os.path.exists(tmp_path / f"ok{r}") for r in range(world))
