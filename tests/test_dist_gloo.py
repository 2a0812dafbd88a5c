"""World-size-2 gloo tests of the multi-GPU path (CPU).

The kernels cannot run here, so the per-rank work is done by the oracle as a
test harness stand-in (never a product fallback); what is tested is the
product's partitioning (dist.shard_views) and its exchange step
(dist.GradBucket: one flat all_reduce of the per-primitive gradients)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_12615_b200 import dist as wdist
from paper_2508_12615_b200 import gen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    c = gen.make_config("p3d", seed=0, N=300, H=48, W=48, B=5)
    views = wdist.shard_views(c["B"], rank, world)
    cams = [c["cams"][v] for v in views]
    cfg = oracle.Cfg(width=48, height=48, prim3d=True, alpha_blend=True,
                     dilation=float(np.float32(0.3)))
    dL = gen.gen_dLdC(c["B"], 48, 48, seed=3)[views]
    dLp = dL.transpose(0, 2, 3, 1).reshape(-1, 3)
    out = oracle.forward_backward(cfg, c["params"], dLp, cams=cams)
    grads = {k: torch.from_numpy(v.astype(np.float32)) for k, v in out["grads"].items()}
    bucket = wdist.GradBucket(grads)
    bucket.all_reduce()
    if rank == 0:
        q.put({k: v.numpy().copy() for k, v in grads.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_shard_views_partition():
    for B in (1, 5, 8, 100):
        for world in (1, 2, 4, 8):
            got = sorted(v for r in range(world) for v in wdist.shard_views(B, r, world))
            assert got == list(range(B))


def test_gradbucket_views_share_storage():
    g = {"a": torch.zeros(3, 2), "b": torch.zeros(5)}
    b = wdist.GradBucket(g)
    g["a"] += 1
    g["b"][2] = 7
    assert b.flat.numel() == 11 and b.flat[:6].sum() == 6 and b.flat[8] == 7


@pytest.mark.timeout(300)
def test_view_sharded_gradients_equal_single_process(ora):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    c = gen.make_config("p3d", seed=0, N=300, H=48, W=48, B=5)
    cfg = ora.Cfg(width=48, height=48, prim3d=True, alpha_blend=True,
                  dilation=float(np.float32(0.3)))
    dL = gen.gen_dLdC(c["B"], 48, 48, seed=3).transpose(0, 2, 3, 1).reshape(-1, 3)
    ref = ora.forward_backward(cfg, c["params"], dL, cams=c["cams"])["grads"]
    for k, v in ref.items():
        np.testing.assert_allclose(got[k], v.astype(np.float32), rtol=1e-5, atol=1e-6)


def _worker_rows(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    H, W = 48, 64
    p = gen.gen2d(H, W, 200, seed=9, freq_std=0.5)
    cfg = oracle.Cfg(width=W, height=H)
    dL = gen.gen_dLdC(1, H, W, seed=9)[0].transpose(1, 2, 0).copy()
    # this rank owns tile rows ty = rank (mod world): only its pixels carry dL/dC
    rows = wdist.tile_rows(-(-H // 16), rank, world)
    mask = np.isin(np.arange(H) // 16, rows)
    dL[~mask] = 0.0
    out = oracle.forward_backward(cfg, p, dL.reshape(-1, 3))
    grads = {k: torch.from_numpy(v.astype(np.float32)) for k, v in out["grads"].items()}
    wdist.GradBucket(grads).all_reduce()
    if rank == 0:
        q.put({k: v.numpy().copy() for k, v in grads.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_tile_row_sharded_gradients_equal_single_process(ora):
    """Image-space sharding: ranks own tile rows ty = r (mod
    world); the all_reduce of their gradients equals the full-image gradient."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_rows, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    H, W = 48, 64
    p = gen.gen2d(H, W, 200, seed=9, freq_std=0.5)
    dL = gen.gen_dLdC(1, H, W, seed=9)[0].transpose(1, 2, 0).reshape(-1, 3)
    ref = ora.forward_backward(ora.Cfg(width=W, height=H), p, dL)["grads"]
    for k, v in ref.items():
        np.testing.assert_allclose(got[k], v.astype(np.float32), rtol=1e-5, atol=1e-6)


def _worker_det(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(100 + rank)
    g = {"a": torch.from_numpy(rng.normal(size=(1000, 3)).astype(np.float32)),
         "b": torch.from_numpy(rng.normal(size=500).astype(np.float32))}
    b = wdist.GradBucket(g, deterministic=True)
    b.all_reduce()
    q.put((rank, {k: v.numpy().copy() for k, v in g.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_deterministic_gradbucket_rank_order_sum():
    """The deterministic all-reduce is the rank-ordered sum, identical on every rank."""
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_det, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    parts = []
    for r in range(world):
        rng = np.random.default_rng(100 + r)
        parts.append({"a": rng.normal(size=(1000, 3)).astype(np.float32),
                      "b": rng.normal(size=500).astype(np.float32)})
    for k in ("a", "b"):
        ref = parts[0][k].copy()
        for r in range(1, world):
            ref += parts[r][k]
        for r in range(world):
            np.testing.assert_array_equal(got[r][k], ref)


def _worker_sets(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    # bench.py's pipelined multi-rank e2e: every buffer set's flat gradient
    # buffer is summed on its own (reduce_flat), in step order
    sets = [torch.full((257,), float(10 * k + rank + 1)) for k in range(3)]
    for k in (0, 1, 2, 0):
        wdist.reduce_flat(sets[k])
    det = torch.arange(100, dtype=torch.float32) * (rank + 1)
    wdist.reduce_flat(det, deterministic=True)
    q.put((rank, [s.numpy().copy() for s in sets], det.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_reduce_flat_per_buffer_set():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_sets, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (s, d)) for r, s, d in (q.get(timeout=240) for _ in range(world)))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(world):
        sets, det = got[r]
        # set 0 reduced twice: (1 + 2) -> 3 + 3; sets 1, 2 once
        assert np.all(sets[0] == 2 * (1 + 2))
        assert np.all(sets[1] == (11 + 12)) and np.all(sets[2] == (21 + 22))
        np.testing.assert_array_equal(det, np.arange(100, dtype=np.float32) * 3)


def test_bench_sharding_modes():
    """bench.py's partitioning per config and world size: C2 is
    one image split by tile rows at N > 1 (replicas only on request), C3 views,
    C4 frames, C5 tile rows."""
    import argparse
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    a = argparse.Namespace(replicas=False)
    assert bench.sharding("c2", 1, a) == (False, False, False)
    assert bench.sharding("c2", 8, a) == (True, False, True)
    assert bench.sharding("c2", 8, argparse.Namespace(replicas=True)) == (False, False, False)
    assert bench.sharding("c3", 8, a) == (False, False, True)
    assert bench.sharding("c4", 8, a) == (False, True, True)
    assert bench.sharding("c5", 1, a) == (True, False, True)


def _worker_rows_bucket(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2508_12615_b200.raster import row_ranges
    rng = np.random.default_rng(40 + rank)
    N = 1000
    g = {"mean": torch.from_numpy(rng.normal(size=(N, 3)).astype(np.float32)),
         "quat": torch.from_numpy(rng.normal(size=(N, 4)).astype(np.float32)),
         "opacity": torch.from_numpy(rng.normal(size=N).astype(np.float32))}
    full = {k: v.clone() for k, v in g.items()}
    for v in full.values():
        dist.all_reduce(v)
    b = wdist.GradBucket(g)
    ov = wdist.OverlappedReduce(b)
    for r0, r1 in row_ranges(N, 3):  # as Rasterizer.backward(row_chunks=3, on_rows=...)
        ov.on_rows(r0, r1)
    ov.finish()
    q.put((rank, {k: v.numpy().copy() for k, v in g.items()},
           {k: v.numpy().copy() for k, v in full.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_bucketed_row_reduce_equals_full_all_reduce():
    """The overlapped exchange (dist.OverlappedReduce / GradBucket.reduce_rows):
    reducing the parameter rows chunk by chunk, every group's slice of each
    chunk, gives exactly the all-reduce of the whole buffers."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_rows_bucket, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for _, chunked, full in got:
        for k in full:
            np.testing.assert_array_equal(chunked[k], full[k])


def test_row_ranges_partition():
    from paper_2508_12615_b200.raster import row_ranges
    for rows in (1, 63, 64, 1000, 1000000):
        for k in (1, 2, 3, 4, 7):
            rr = row_ranges(rows, k)
            assert rr[0][0] == 0 and rr[-1][1] == rows
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(rr, rr[1:]))
            assert all(r0 % 64 == 0 for r0, _ in rr)
