"""Multi-GPU host logic on CPU (gloo, world size 2 and 4): light layout,
Gaussian shards, partial-tau reduce-scatter over K + exp epilogue, and the
product-over-lights query combine (paper_2601_01660_b200/distributed.py).

The per-rank build is the CPU oracle here (this box has no GPU); the
collective structure is exactly the one the CUDA path runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_01660_b200 import distributed as D
from paper_2601_01660_b200 import synth


def test_plan_layout_light_parallel():
    lay = D.plan_layout(8, 4, light_cost=[8, 7, 6, 5, 4, 3, 2, 1])
    assert lay.groups == [[0], [1], [2], [3]]
    assert sorted(sum(lay.lights_of, [])) == list(range(8))
    loads = [sum(8 - l for l in ls) for ls in lay.lights_of]
    assert max(loads) - min(loads) <= 1  # LPT balances 8..1 over 4 ranks perfectly
    lay = D.plan_layout(4, 4)
    assert lay.lights_of == [[0], [1], [2], [3]]


def test_plan_layout_gaussian_sharded():
    lay = D.plan_layout(1, 8)
    assert lay.groups == [list(range(8))] and lay.lights_of == [[0]]
    lay = D.plan_layout(3, 8)
    assert [len(g) for g in lay.groups] == [3, 3, 2]
    assert sorted(sum(lay.groups, [])) == list(range(8))
    assert lay.shard_of(4) == (1, 3)


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 1001):
        for g in (1, 2, 3, 8):
            rs = [D.shard_range(n, i, g) for i in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_build_fn(g_t, lights, res, K, output_tau=False):
    from oracle import oracle
    g = {k: v.numpy() for k, v in g_t.items()}
    T, _ = oracle.build(g, lights, res, K, n_threads=2)
    out = -np.log(T) if output_tau else T
    return torch.from_numpy(out.astype(np.float32))


def oracle_query_fn(atlas, lights, positions):
    from oracle import oracle
    return torch.from_numpy(oracle.query(atlas.numpy().astype(np.float64), lights, positions.numpy()).astype(np.float32))


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "gaussian":
            s = synth.config1()
            s = synth.Scene("c", {k: v[:400] for k, v in s.gaussians.items()}, s.lights, 32, 8, s.queries[:300])
        else:
            s = synth.random_scene(3, 200, res=16, K=4, L=3, dist=(0.5, 3.0))
        g = {k: torch.from_numpy(v) for k, v in s.gaussians.items()}
        lay = D.plan_layout(s.L, world)
        pg = D.make_groups(lay)
        atl = D.build_sharded(g, s.lights, s.res, s.K, lay, pg, oracle_build_fn, lambda t: torch.exp(-t))
        T = D.query_sharded(atl, s.lights, torch.from_numpy(s.queries), lay, oracle_query_fn)
        q.put((rank, {l: a.numpy() for l, a in atl.items()}, T.numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def _reference(case):
    from oracle import oracle
    if case == "gaussian":
        s = synth.config1()
        s = synth.Scene("c", {k: v[:400] for k, v in s.gaussians.items()}, s.lights, 32, 8, s.queries[:300])
    else:
        s = synth.random_scene(3, 200, res=16, K=4, L=3, dist=(0.5, 3.0))
    T, _ = oracle.build(s.gaussians, s.lights, s.res, s.K)
    Tf = T.astype(np.float32).astype(np.float64)
    return s, T, oracle.query(Tf, s.lights, s.queries)


@pytest.mark.parametrize("world", [2, 4])
def test_gaussian_sharded_reduce_scatter(world):
    """1 light on `world` ranks: partial tau per Gaussian shard, reduce-scatter
    over K, exp on the owned shells, all-gather == unsharded oracle atlas."""
    res = _run(world, "gaussian")
    s, T, Tq = _reference("gaussian")
    for rank, atl, Tr in res:
        assert list(atl) == [0]
        assert np.abs(atl[0] - T[0]).max() < 2e-6
        assert np.abs(Tr - Tq).max() < 2e-6


def test_light_parallel_query_product():
    """3 lights on 2 ranks (light-parallel, no build communication); the query
    product over lights is an all-reduce(PRODUCT)."""
    res = _run(2, "lights")
    s, T, Tq = _reference("lights")
    owned = {}
    for rank, atl, Tr in res:
        for l, a in atl.items():
            owned[l] = a
        assert np.abs(Tr - Tq).max() < 1e-5
    assert sorted(owned) == [0, 1, 2]
    for l, a in owned.items():
        assert np.abs(a - T[l]).max() < 1e-6
