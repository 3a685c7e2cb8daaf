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
    every image's descriptors. `local` maps image index -> uint8 (M_i, B) array (numpy or
    torch) for the images this rank extracted (image i lives on rank i mod world, as
    extract_images_sharded deals them). One all_reduce of the row counts and ONE padded
    all_gather_into_tensor of the rank's rows (131 MB in total at cfg5) — not a broadcast per
    image. Returns a list of num_images uint8 torch tensors on `device` (the rank's GPU under
    NCCL, CPU under gloo); entry i is a view into the gathered block."""
    import torch
    dist = _dist()
    rank, world = _world()
    device = device or torch.device("cpu")
    nbytes = next((int(v.shape[1]) for v in local.values()), 64)
    counts = torch.zeros(num_images, dtype=torch.int64, device=device)
    for i, d in local.items():
        counts[i] = len(d)
    if world > 1:
        dist.all_reduce(counts)                       # each image is owned by exactly one rank
    counts = counts.cpu().tolist()
    owned = [list(range(r, num_images, world)) for r in range(world)]
    rows_of = [sum(counts[i] for i in owned[r]) for r in range(world)]
    cap = max(max(rows_of), 1)
    mine = torch.zeros((cap, nbytes), dtype=torch.uint8, device=device)
    at = 0
    for i in owned[rank]:
        if counts[i]:
            mine[at:at + counts[i]] = torch.as_tensor(np.ascontiguousarray(local[i]) if isinstance(local[i], np.ndarray)
                                                      else local[i], device=device)
        at += counts[i]
    if world > 1:
        flat = torch.empty((world * cap, nbytes), dtype=torch.uint8, device=device)
        dist.all_gather_into_tensor(flat, mine)       # rank r's rows land at [r * cap, (r + 1) * cap)
        block = flat.view(world, cap, nbytes)
    else:
        block = mine.unsqueeze(0)
    sets = [None] * num_images
    for r in range(world):
        at = 0
        for i in owned[r]:
            sets[i] = block[r, at:at + counts[i]]
            at += counts[i]
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
    q_total = queries.shape[0]
    begin, end = shard_bounds(q_total, world)[rank]
    if gather:
        return match_top2_sharded_device(queries[begin:end], train, q_total, train_src, top2)
    if world > 1:
        dist.broadcast(train, src=train_src)          # the single large message (N x 64 B)
    local = top2(queries[begin:end], train) if end > begin else \
        torch.empty((3, 0), dtype=torch.int32, device=queries.device)
    return local, (begin, end)


def match_all_pairs_sharded(desc_sets: Sequence, match_pair: Callable, num_images: int | None = None):
    """cfg5: exhaustive pairwise matching. `match_pair(i, j, desc_i, desc_j)` returns the
    matches of image pair (i, j) (any object; typically an (M,4) int32 array). Returns
    {(i, j): result} for the pairs this rank owns."""
    rank, world = _world()
    n = num_images if num_images is not None else len(desc_sets)
    return {(i, j): match_pair(i, j, desc_sets[i], desc_sets[j]) for i, j in pairs_for_rank(n, rank, world)}


def match_all_pairs_resident(desc_sets: Sequence, ratio=None, cross_check=False, max_distance=None,
                             num_images: int | None = None, resident: dict | None = None):
    """cfg5 on the CUDA path: this rank's share of the (i < j) pairs, batched through resident
    descriptor sets (each image is uploaded and expanded once, all pairs run in a few launches).
    `desc_sets[i]` is a (M_i, 64) uint8 numpy array or CUDA tensor; `resident` (from
    create_resident_sets) skips the upload when the sets already live on the device.
    Returns {(i, j): (M,4) int32}."""
    from .engine import get_engine
    rank, world = _world()
    n = num_images if num_images is not None else len(desc_sets)
    mine = pairs_for_rank(n, rank, world)
    if not mine:
        return {}
    eng = get_engine()
    needed = sorted({i for p in mine for i in p})
    sets = resident if resident is not None else {i: eng.create_set(desc_sets[i]) for i in needed}
    order = {i: k for k, i in enumerate(needed)}
    try:
        res = eng.match_set_pairs([sets[i] for i in needed], [(order[i], order[j]) for i, j in mine],
                                  ratio=ratio, cross_check=cross_check, max_distance=max_distance)
    finally:
        if resident is None:
            for s in sets.values():
                s.close()
    return dict(zip(mine, res))          # views into one result block


def create_resident_sets(desc_sets: Sequence, num_images: int | None = None) -> dict:
    """Device-resident sets {image index: DescriptorSet} for the images this rank's pairs touch."""
    from .engine import get_engine
    rank, world = _world()
    n = num_images if num_images is not None else len(desc_sets)
    needed = sorted({i for p in pairs_for_rank(n, rank, world) for i in p})
    eng = get_engine()
    return {i: eng.create_set(desc_sets[i]) for i in needed}


def match_sharded_host(queries: np.ndarray, train: np.ndarray, ratio=None, max_distance=None, train_src: int = 0):
    """cfg4 end to end from HOST arrays: rank `train_src` uploads the train set and broadcasts it
    over NCCL, every rank uploads only its own query block, matches it, and the (3, Q) top-2
    triples are all-gathered; the reference's filter pass (src/match.cpp:69-79, ratio / max
    distance) then runs on the gathered triples. Returns (M, 4) int32 rows like match()."""
    import torch
    from .engine import get_engine
    rank, world = _world()
    eng = get_engine()
    dev = torch.device("cuda", eng.device)
    q_total = len(queries)
    begin, end = shard_bounds(q_total, world)[rank]
    if world == 1:
        bi, bd, sd = eng.match_top2(queries, train)
    else:
        d_train = torch.empty(train.shape, dtype=torch.uint8, device=dev)
        if rank == train_src:
            d_train.copy_(torch.from_numpy(train))
        d_q = torch.from_numpy(np.ascontiguousarray(queries[begin:end])).to(dev)
        full = match_top2_sharded_device(d_q, d_train, q_total, train_src).cpu().numpy()
        bi, bd, sd = full[0], full[1], full[2]
    return eng.filter_matches(bi, bd, sd, ratio=ratio, max_distance=max_distance)


def match_top2_sharded_device(q_shard, train, q_total: int, train_src: int = 0, top2: Callable = default_top2):
    """The collective part of cfg4 on device tensors: `q_shard` holds this rank's contiguous query
    block (shard_bounds(q_total, world)[rank]), `train` is valid on `train_src` and is broadcast in
    place; returns the full (3, q_total) int32 result on every rank."""
    import torch
    dist = _dist()
    rank, world = _world()
    if world > 1:
        dist.broadcast(train, src=train_src)
    local = top2(q_shard, train) if q_shard.shape[0] else torch.empty((3, 0), dtype=torch.int32, device=train.device)
    if world == 1:
        return local
    chunk = (q_total + world - 1) // world
    padded = torch.zeros((3, chunk), dtype=torch.int32, device=train.device)
    padded[:, :local.shape[1]] = local
    flat = torch.empty((world * 3, chunk), dtype=torch.int32, device=train.device)
    dist.all_gather_into_tensor(flat, padded)             # 12 B per query
    return flat.view(world, 3, chunk).permute(1, 0, 2).reshape(3, world * chunk)[:, :q_total].contiguous()


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
