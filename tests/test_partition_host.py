"""Host logic of the row partition, CPU only.

* the plan every rank computes (sk_partition_plan): contiguous, covering,
  chunk-aligned, balanced, every rank >= the operator halo;
* the reduction contract it relies on, exercised across two real processes
  (gloo, world_size 2): each rank reduces only its own rows into chunk nodes
  (the R1 contract on its rows, zeros elsewhere), the nodes are all-gathered,
  and the canonical pairwise tree over them in global order is bitwise the
  single-process R1 reduction (oracle sko_r1_dot).
"""
import os
import socket
import struct

import numpy as np
import pytest


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def tree(vals):
    """Canonical pairwise tree (adjacent pairs, odd tail passes through)."""
    a = list(vals)
    if not a:
        return 0.0
    while len(a) > 1:
        a = [a[i] + a[i + 1] if i + 1 < len(a) else a[i] for i in range(0, len(a), 2)]
    return a[0]


@pytest.mark.parametrize("n,halo", [(65536, 256), (16777216, 4096), (4096 * 4096 + 12345, 4096),
                                    (2097152, 16384), (300000, 300)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_properties(sk_host, n, halo, world):
    sk = sk_host
    try:
        plans = [sk.partition_plan(n, halo, world, r) for r in range(world)]
    except sk.UnsupportedError:
        assert n < 16384 * world or n // world < halo * 2
        return
    cr = plans[0]["chunk_rows"]
    assert cr % 16384 == 0 and (cr // 512) & (cr // 512 - 1) == 0  # power-of-two segments >= 32
    pos = 0
    for p in plans:
        assert p["row0"] == pos and p["row0"] % cr == 0
        assert p["rows"] > 0 and (world == 1 or p["rows"] >= halo)
        assert p["chunks"] == -(-p["rows"] // cr)
        assert p["chunks_max"] == max(q["chunks"] for q in plans)
        pos += p["rows"]
    assert pos == n
    assert sum(p["chunks"] for p in plans) == plans[0]["chunks_total"]
    counts = [p["chunks"] for p in plans]
    assert max(counts) - min(counts) <= 1
    assert plans[0]["halo"] == (halo if world > 1 else 0)


def _worker(rank, world, port, n, out_dir):
    import torch.distributed as dist
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.join(here, "..")]
    import paper_2605_28274_b200 as sk
    from oracle import pyoracle as po

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(2024)
    x = rng.standard_normal(n)
    y = rng.standard_normal(n)
    plan = sk.partition_plan(n, 0, world, rank)
    nodes = []
    for j in range(plan["chunks"]):
        lo = plan["row0"] + j * plan["chunk_rows"]
        hi = min(lo + plan["chunk_rows"], plan["row0"] + plan["rows"])
        xm = np.zeros(n)
        xm[lo:hi] = x[lo:hi]  # this rank sees only its rows
        nodes.append(po.r1_dot(xm, y))
    gathered = [None] * world
    dist.all_gather_object(gathered, nodes)
    root = tree([v for r in range(world) for v in gathered[r]])
    full = po.r1_dot(x, y)
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
        f.write(f"{struct.pack('<d', root).hex()} {struct.pack('<d', full).hex()}\n")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [65536 + 1000, 3 * 16384])
def test_chunk_nodes_compose_across_processes(tmp_path, n):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        root, full = open(tmp_path / f"rank{r}.txt").read().split()
        assert root == full, f"rank {r}: partitioned root {root} != single-process {full}"


def test_single_rank_tree_matches_oracle_r1(po):
    """Sanity: chunk nodes of one process compose to the oracle's R1 reduction."""
    n = 100000
    rng = np.random.default_rng(7)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    cr = 32 * 512
    nodes = []
    for lo in range(0, n, cr):
        xm = np.zeros(n)
        xm[lo:lo + cr] = x[lo:lo + cr]
        nodes.append(po.r1_dot(xm, y))
    assert struct.pack("<d", tree(nodes)) == struct.pack("<d", po.r1_dot(x, y))
