"""Multi-GPU partitioning host logic on CPU: world_size-2 (and 3) gloo runs of
the halo exchange, checked against the unsharded signal, and the sharded
outputs recomputed by the oracle from each rank's halo'd buffer only."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1910_01972_b200 as oc
from paper_1910_01972_b200.sharding import (HaloBuffer, exchange_halos,
                                            make_shards)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [
    (20000, 400, 3, 2048, 0),
    (9000, 129, 2, 1024, 64),
    (5000, 33, 2, 128, 16),
    (700, 64, 1, 64, 63),
]


@pytest.mark.parametrize("mode", ["c2c", "r2r"])
def test_shards_partition_and_cover_dependencies(mode):
    for ns, m, nfil, n, origin in CASES:
        p = oc.plan(ns, m, mode, origin, n)
        for world in (1, 2, 3, 8, 64):
            sh = make_shards(p, world)
            assert len(sh) == world
            cov = np.zeros(ns, int)
            for s in sh:
                cov[s.g_lo:s.g_hi] += 1
                if s.g_hi > s.g_lo:
                    # inputs of outputs [g_lo, g_hi): [g_lo-(m-1)+o, g_hi+o)
                    need_lo = max(0, s.g_lo - (m - 1) + origin)
                    need_hi = min(ns, s.g_hi + origin)
                    assert s.x_lo <= need_lo and s.x_hi >= need_hi
                    assert s.left_halo >= 0 and s.right_halo >= 0
            assert np.all(cov == 1), (ns, m, world)
            # the derivative's shards also cover the neighbours' inputs
            if n - m - 1 >= 1:
                for s in make_shards(p, world,
                                     postproc=oc.PostProcSpec("derivative")):
                    if s.g_hi > s.g_lo:
                        need_lo = max(0, s.g_lo - 1 - (m - 1) + origin)
                        need_hi = min(ns, s.g_hi + 1 + origin)
                        assert s.x_lo <= need_lo and s.x_hi >= need_hi


def _worker(rank, world, port, case, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        ns, m, nfil, n, origin = case
        rng = np.random.default_rng([7, ns, m])
        x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
        taps = rng.standard_normal((nfil, m)) + 1j * rng.standard_normal((nfil, m))
        p = oc.plan(ns, m, "c2c", origin, n)
        shards = make_shards(p, world)
        me = shards[rank]
        own = torch.from_numpy(x[me.g_lo:me.g_hi].copy())
        buf = exchange_halos(own, shards, rank)
        ok_buf = np.array_equal(buf.numpy(), x[me.x_lo:me.x_hi])
        # this rank's outputs from its halo'd buffer alone (oracle, fp64):
        # embed the buffer in zeros, i.e. no sample outside [x_lo, x_hi)
        if me.g_hi > me.g_lo:
            sub = np.zeros(ns, np.complex128)
            sub[me.x_lo:me.x_hi] = buf.numpy()
            y = oracle.direct_window(sub, taps, origin, me.g_lo, me.g_hi, 2)
            ref = oracle.direct_window(x, taps, origin, me.g_lo, me.g_hi, 2)
            err = float(np.max(np.abs(y - ref)))
        else:
            err = 0.0
        ret[rank] = (ok_buf, err)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_gloo_halo_exchange(world, case):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES[case], ret))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    for r in range(world):
        ok_buf, err = ret[r]
        assert ok_buf, r
        assert err == 0.0, (r, err)


def _worker_halo_buffer(rank, world, port, case, ret):
    """Persistent halo'd buffer: owned samples written once, every step moves
    only the halos.  Two steps with new owned data; after each exchange the
    buffer equals the global signal over [x_lo, x_hi)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ns, m, nfil, n, origin = case
        p = oc.plan(ns, m, "c2c", origin, n)
        shards = make_shards(p, world)
        me = shards[rank]
        hb = HaloBuffer(shards, rank, torch.complex128, "cpu")
        ok = []
        moved = hb.halo_samples
        for step in range(2):
            rng = np.random.default_rng([8, step, ns, m])
            x = rng.standard_normal(ns) + 1j * rng.standard_normal(ns)
            hb.own.copy_(torch.from_numpy(x[me.g_lo:me.g_hi]))
            buf = hb.exchange()
            ok.append(np.array_equal(buf.numpy()[:me.x_hi - me.x_lo],
                                     x[me.x_lo:me.x_hi]))
        ret[rank] = (all(ok), moved, (me.g_lo - me.x_lo) + (me.x_hi - me.g_hi))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_gloo_persistent_halo_buffer(world, case):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker_halo_buffer,
                         args=(r, world, port, CASES[case], ret))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    for r in range(world):
        ok, moved, halo = ret[r]
        assert ok, r
        assert moved == halo, (r, moved, halo)   # only the halos move
