"""world_size-2 gloo tests (CPU) of the multi-GPU host logic in sharded.py: partitioning,
the train-set broadcast, the top-2 gather, the descriptor all-gather and pair dealing.
The per-rank compute step is injected (the CPU oracle stands in for the CUDA kernels —
this is the checker used as a stub inside a test, never the product path)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist            # noqa: E402
import torch.multiprocessing as mp          # noqa: E402

from paper_1609_03986_b200 import sharded   # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_top2(queries, train):
    import oracle
    r = oracle.port().knn2_all(queries.numpy(), train.numpy())
    return torch.from_numpy(np.ascontiguousarray(r.T))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    po = oracle.port()
    try:
        # ---- cfg4 shape: query shards + train broadcast + top-2 gather ----
        q = torch.from_numpy(po.random_descriptors(41, 301, 64))
        train_np = po.random_descriptors(42, 257, 64)
        train_np[200] = train_np[3]
        q[5] = torch.from_numpy(train_np[3])
        train = torch.from_numpy(train_np) if rank == 0 else torch.zeros((257, 64), dtype=torch.uint8)
        got = sharded.match_top2_sharded(q, train, top2=_oracle_top2)
        want = po.knn2_all(q.numpy(), train_np).T
        assert np.array_equal(got.numpy(), want), "gathered top-2 differs"
        assert np.array_equal(train.numpy(), train_np), "train set was not broadcast"
        local, (b, e) = sharded.match_top2_sharded(q, train, top2=_oracle_top2, gather=False)
        assert (b, e) == sharded.shard_bounds(301, world)[rank]
        assert np.array_equal(local.numpy(), want[:, b:e])

        # ---- cfg3 + cfg5 shape: images by rank, all-gather, pairs by rank ----
        num_images = 5
        sets_np = [po.random_descriptors(100 + i, 20 + 3 * i, 64) for i in range(num_images)]
        mine = sharded.extract_images_sharded(list(range(num_images)), list(range(num_images)),
                                              describe=lambda img, kps: (None, sets_np[img]))
        assert sorted(mine) == list(range(rank, num_images, world))
        sets = sharded.all_gather_descriptor_sets({i: v[1] for i, v in mine.items()}, num_images)
        for i in range(num_images):
            assert np.array_equal(sets[i].numpy(), sets_np[i]), f"descriptor set {i} differs after all_gather"
        res = sharded.match_all_pairs_sharded(
            sets, lambda i, j, a, b: po.match(a.numpy(), b.numpy(), ratio=0.9, cross_check=True))
        assert sorted(res) == sharded.pairs_for_rank(num_images, rank, world)
        for (i, j), m in res.items():
            assert np.array_equal(m, po.match(sets_np[i], sets_np[j], ratio=0.9, cross_check=True))
        counts = torch.tensor([len(res)])
        dist.all_reduce(counts)
        assert counts.item() == num_images * (num_images - 1) // 2      # every pair exactly once
        out.put((rank, "ok"))
    except Exception as exc:                                            # noqa: BLE001
        out.put((rank, f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


def test_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(out.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results


def test_partition_rules():
    assert sharded.shard_bounds(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert sharded.shard_bounds(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert sharded.shard_bounds(0, 2) == [(0, 0), (0, 0)]
    for n, w in ((1_000_000, 8), (125, 8), (7, 8)):
        b = sharded.shard_bounds(n, w)
        assert b[0][0] == 0 and b[-1][1] == n and all(x[1] == y[0] for x, y in zip(b, b[1:]))
    allp = [p for r in range(8) for p in sharded.pairs_for_rank(256, r, 8)]
    assert len(allp) == len(set(allp)) == 256 * 255 // 2          # cfg5: 32 640 pairs, each once
    sizes = [len(sharded.pairs_for_rank(256, r, 8)) for r in range(8)]
    assert max(sizes) - min(sizes) <= 1
    # single process, no process group: world of one
    q = torch.zeros((4, 64), dtype=torch.uint8)
    t = torch.zeros((3, 64), dtype=torch.uint8)
    got = sharded.match_top2_sharded(q, t, top2=_oracle_top2)
    assert got.shape == (3, 4) and got[0].tolist() == [0, 0, 0, 0]
