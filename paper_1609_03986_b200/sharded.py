"""Multi-GPU drivers: one process per GPU, torch.distributed for the plumbing.

Both hot paths shard over independent units, so no collective sits
inside a kernel's critical path:

  extraction      by image (cfg3): image i -> rank i mod world; nothing is exchanged
                  unless matching follows, then one all_gather of descriptor shards
  single match    by query block (cfg4): the train set is broadcast once from its
                  owner (NCCL over NVLink/NVSwitch), each rank matches its contiguous
                  query shard against the full train set, only the top-2 triples
                  (12 B per query) are gathered
  all-pairs       by image pair (cfg5): the (i < j) pairs are dealt round-robin; every
                  rank holds all descriptor sets (after the all_gather above)

The reference has no counterpart (single process, std::thread fan-out,
proj/src/parallel.hpp:17-38); the partitioning mirrors its "contiguous chunks, one
output slot per index" rule so results are independent of the world size.

Every function takes the per-rank compute step as a callable so the host-side logic
(partitioning, exchange, ordering) is testable on CPU with the gloo backend; the
default callables run the CUDA kernels through `Engine`.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, near-equal [begin, end) per rank — parallel_for's chunking rule
    (proj/src/parallel.hpp:29-33): chunk = ceil(n / world)."""
    chunk = (n + world - 1) // world if world > 0 else n
    return [(min(n, r * chunk), min(n, (r + 1) * chunk)) for r in range(world)]


def pairs_for_rank(num_images: int, rank: int, world: int) -> list[tuple[int, int]]:
    """The (i < j) image pairs of an exhaustive SfM-style matching job owned by `rank`
    (round-robin over the row-major pair list)."""
    pairs = [(i, j) for i in range(num_images) for j in range(i + 1, num_images)]
    return pairs[rank::world]


def _dist():
    import torch.distributed as dist
    return dist


def _world():
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


# ------------------------------------------------------------------ extraction ----

def extract_images_sharded(images: Sequence, keypoints: Sequence, describe: Callable | None = None):
    """cfg3: images[i] is processed by rank i mod world. `describe(image, keypoints) ->
    (kept, descriptors)`; default = the package's describe(). Returns {image index:
    (kept, descriptors)} for the images this rank owns."""
    rank, world = _world()
    mine = list(range(rank, len(images), world))
    if describe is None:      # CUDA path: this rank's images through one pipelined batch call
        from . import describe_batch
        return dict(zip(mine, describe_batch([images[i] for i in mine], [keypoints[i] for i in mine])))
    return {i: describe(images[i], keypoints[i]) for i in mine}


def all_gather_descriptor_sets(local: dict, num_images: int, device=None):
    """The one exchange step before all-pairs matching (cfg5): every rank ends up with
    every image's descriptors. `local` maps image index -> uint8 (M_i, B) array for the
    images this rank extracted. Returns a list of num_images uint8 torch tensors on
    `device` (the rank's GPU under NCCL, CPU under gloo)."""
    import torch
    dist = _dist()
    rank, world = _world()
    device = device or torch.device("cpu")
    nbytes = next((v.shape[1] for v in local.values()), 64)
    counts = torch.zeros(num_images, dtype=torch.int64, device=device)
    for i, d in local.items():
        counts[i] = len(d)
    if world > 1:
        dist.all_reduce(counts)                       # each image is owned by exactly one rank
    sets = []
    for i in range(num_images):
        owner = i % world
        if i in local:
            t = torch.as_tensor(np.ascontiguousarray(local[i]), device=device)
        else:
            t = torch.empty((int(counts[i]), nbytes), dtype=torch.uint8, device=device)
        if world > 1:
            dist.broadcast(t, src=owner)
        sets.append(t)
    return sets


# -------------------------------------------------------------------- matching ----

def default_top2(queries, train):
    """(Q,B),(N,B) CUDA uint8 tensors -> int32 CUDA tensor (3,Q) via the CUDA matcher."""
    from .engine import get_engine
    return get_engine(queries.device.index).match_top2_device(queries.contiguous(), train.contiguous())


def match_top2_sharded(queries, train, top2: Callable = default_top2, train_src: int = 0,
                       gather: bool = True):
    """cfg4: one large match. `queries` (Q,B) is the FULL query set (every rank passes the
    same tensor or at least the same shape; only the rank's shard is read); `train` (N,B)
    must be valid on `train_src` and is broadcast to the others in place. Returns the full
    (3,Q) int32 result [best_idx, best_dist, second_dist] on every rank when `gather`,
    else this rank's shard and its (begin, end)."""
    import torch
    dist = _dist()
    rank, world = _world()
    if world > 1:
        dist.broadcast(train, src=train_src)          # the single large message (N x 64 B)
    q_total = queries.shape[0]
    begin, end = shard_bounds(q_total, world)[rank]
    local = top2(queries[begin:end], train) if end > begin else \
        torch.empty((3, 0), dtype=torch.int32, device=queries.device)
    if not gather:
        return local, (begin, end)
    if world == 1:
        return local
    chunk = (q_total + world - 1) // world
    padded = torch.zeros((3, chunk), dtype=torch.int32, device=queries.device)
    padded[:, :end - begin] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded)                    # 12 B per query
    return torch.cat(parts, dim=1)[:, :q_total].contiguous()


def match_all_pairs_sharded(desc_sets: Sequence, match_pair: Callable, num_images: int | None = None):
    """cfg5: exhaustive pairwise matching. `match_pair(i, j, desc_i, desc_j)` returns the
    matches of image pair (i, j) (any object; typically an (M,4) int32 array). Returns
    {(i, j): result} for the pairs this rank owns."""
    rank, world = _world()
    n = num_images if num_images is not None else len(desc_sets)
    return {(i, j): match_pair(i, j, desc_sets[i], desc_sets[j]) for i, j in pairs_for_rank(n, rank, world)}


def match_all_pairs_resident(desc_sets: Sequence, ratio=None, cross_check=False, max_distance=None,
                             num_images: int | None = None):
    """cfg5 on the CUDA path: this rank's share of the (i < j) pairs, batched through resident
    descriptor sets (each image is uploaded and expanded once, all pairs run in a few launches).
    `desc_sets[i]` is a (M_i, 64) uint8 numpy array or CUDA tensor. Returns {(i, j): (M,4) int32}."""
    from .engine import get_engine
    rank, world = _world()
    n = num_images if num_images is not None else len(desc_sets)
    mine = pairs_for_rank(n, rank, world)
    eng = get_engine()
    needed = sorted({i for p in mine for i in p})
    sets = {i: eng.create_set(desc_sets[i]) for i in needed}
    order = {i: k for k, i in enumerate(needed)}
    try:
        res = eng.match_set_pairs([sets[i] for i in needed], [(order[i], order[j]) for i, j in mine],
                                  ratio=ratio, cross_check=cross_check, max_distance=max_distance)
    finally:
        for s in sets.values():
            s.close()
    return dict(zip(mine, res))          # views into one result block


def default_match_pair(ratio=None, cross_check=False, max_distance=None):
    """match_pair callable for match_all_pairs_sharded running the CUDA matcher on device
    tensors and the reference's filter pass on the host (src/match.cpp:69-79)."""
    from .engine import get_engine

    def run(i, j, di, dj):
        import torch
        eng = get_engine(di.device.index)
        fwd = eng.match_top2_device(di, dj)
        rev = eng.match_top2_device(dj, di)[0] if cross_check else None
        torch.cuda.current_stream(di.device).synchronize()
        f = fwd.cpu().numpy()
        return eng.filter_matches(f[0], f[1], f[2], ratio=ratio, max_distance=max_distance,
                                  reverse_best=None if rev is None else rev.cpu().numpy())
    return run
