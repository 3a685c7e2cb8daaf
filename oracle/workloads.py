"""TEST INFRASTRUCTURE — the five BASELINE.json configurations as seeded synthetic inputs.

Everything is drawn with the reference's own generator (latch::Rng restated in
oracle/latch_oracle.c, checked against the reference in tests/test_oracle.py), with the
seeds SURVEY.md §8(d) fixes, so the CUDA path, the C restatement and the compiled reference
all see the same bytes. Used by tests/, bench.py (input synthesis and the CPU baseline) and
nothing in the product package.

    cfg1  640x480 u8 noise image, 2 000 oriented keypoints, extract + 2k x 2k top-2 self-match
    cfg2  1920x1080, 10 000 keypoints, extract + 10k x 10k
    cfg3  64 images 3840x2160 x 50 000 keypoints each, extraction sharded by image
    cfg4  1 M x 1 M 64-byte descriptors, ratio test 0.8, train set broadcast, queries sharded
    cfg5  256 images 1920x1080 x 8 000 keypoints, all 32 640 image pairs (ratio 0.8 + cross-check)
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import cpu_threads, port

# name -> (width, height, keypoints per image, image seed, keypoint seed, images)
IMAGE_CONFIGS = {
    "cfg1": (640, 480, 2000, 1609, 1610, 1),
    "cfg2": (1920, 1080, 10000, 3986, 3987, 1),
    "cfg3": (3840, 2160, 50000, 30000, 31000, 64),
    "cfg5": (1920, 1080, 8000, 50000, 51000, 256),
}
CFG4_ROWS = 1_000_000
CFG4_QUERY_SEED, CFG4_TRAIN_SEED = 41, 42
RATIO = 0.8

DESCRIPTIONS = {
    "cfg1": "cfg1: 640x480 u8 noise image, 2000 oriented keypoints, extract + 2000x2000 Hamming top-2 self-match",
    "cfg2": "cfg2: 1920x1080 u8 noise image, 10000 oriented keypoints, extract + 10000x10000 Hamming top-2 self-match",
    "cfg3": "cfg3: 64 u8 noise images 3840x2160 x 50000 oriented keypoints each, extraction sharded by image",
    "cfg4": "cfg4: 1000000 x 1000000 64-byte descriptors (1% planted copies, 0.1% duplicated train rows), top-2 + "
            "ratio test 0.8, train set broadcast, queries sharded",
    "cfg5": "cfg5: 256 u8 noise images 1920x1080 x 8000 keypoints, all 32640 image pairs matched with ratio 0.8 + "
            "cross-check, pairs sharded",
}


def image(cfg: str, i: int = 0, rank_offset: int = 0) -> np.ndarray:
    """u8 noise image i of an image configuration (testutil::random_image, integer valued)."""
    w, h, _, s_img, _, count = IMAGE_CONFIGS[cfg]
    assert 0 <= i < count
    return port().random_image_u8(s_img + i + 1000 * rank_offset, w, h)


def keypoints(cfg: str, i: int = 0, rank_offset: int = 0) -> np.ndarray:
    """(n, 4) float64 [x, y, theta, 0]: uniform inside the 46 px margin, theta uniform in [-pi, pi)
    (the recipe of proj/tests/acceptance.cpp:43-49)."""
    w, h, n, _, s_kp, count = IMAGE_CONFIGS[cfg]
    assert 0 <= i < count
    return port().random_keypoints(s_kp + i + 1000 * rank_offset, w, h, n)


def images_and_keypoints(cfg: str, indices, threads: int | None = None):
    """Many images of one configuration, generated on all host threads (ctypes drops the GIL)."""
    indices = list(indices)
    with ThreadPoolExecutor(threads or cpu_threads()) as ex:
        imgs = list(ex.map(lambda i: image(cfg, i), indices))
        kps = list(ex.map(lambda i: keypoints(cfg, i), indices))
    return imgs, kps


def cfg4_sets(rows: int = CFG4_ROWS, train_rows: int | None = None):
    """(queries, train, planted): uniform random descriptors (testutil::random_descriptor) with the
    structure of proj/tests/acceptance.cpp:170-173 — 0.1 % of the train rows are duplicates of other
    train rows (ties: the lowest index must win) and 1 % of the queries are exact copies of train rows
    (distance 0). `planted` = (query rows, the train rows they were copied from)."""
    n = rows if train_rows is None else train_rows
    p = port()
    q = p.random_descriptors(CFG4_QUERY_SEED, rows, 64)
    t = p.random_descriptors(CFG4_TRAIN_SEED, n, 64)
    rng = np.random.default_rng(4)
    dup_t = rng.choice(n, max(n // 1000, 1), replace=False)
    t[dup_t] = t[(dup_t * 7 + 3) % n]                       # duplicated train rows first ...
    dup_q = rng.choice(rows, max(rows // 100, 1), replace=False)
    src_t = rng.integers(0, n, len(dup_q))
    q[dup_q] = t[src_t]                                     # ... then copies of the final train rows
    return q, t, (dup_q, src_t)


def all_pairs(num_images: int):
    return [(i, j) for i in range(num_images) for j in range(i + 1, num_images)]


# ---- threaded front-ends of the serial C restatement (for at-size parity samples) ----

def knn2_rows_threaded(probes: np.ndarray, gallery: np.ndarray, threads: int | None = None) -> np.ndarray:
    """oracle knn2 of every probe row against the gallery -> int32 (Q, 3), on all host threads."""
    p = port()
    threads = threads or cpu_threads()
    bounds = np.linspace(0, len(probes), threads + 1).astype(int)
    out = np.zeros((len(probes), 3), np.int32)

    def work(k):
        b, e = int(bounds[k]), int(bounds[k + 1])
        if e > b:
            out[b:e] = p.knn2_all(probes[b:e], gallery)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return out


def describe_all_threaded(img: np.ndarray, kps: np.ndarray, threads: int | None = None):
    """oracle describe_all on all host threads -> (kept indices, descriptors), input order."""
    p = port()
    threads = threads or cpu_threads()
    img = np.ascontiguousarray(img, np.float64)
    bounds = np.linspace(0, len(kps), threads + 1).astype(int)

    def work(k):
        b, e = int(bounds[k]), int(bounds[k + 1])
        kept, desc = p.describe_all(img, kps[b:e])
        return kept + b, desc
    with ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(work, range(threads)))
    return np.concatenate([a for a, _ in parts]), np.concatenate([d for _, d in parts])


def match_threaded(probes, gallery, ratio=None, cross_check=False, max_distance=None, threads: int | None = None):
    """oracle match_brute_force (src/match.cpp:52-81) with the two knn2 passes on all host threads and
    the serial filter pass of the C restatement's rule set, restated here in numpy order."""
    fwd = knn2_rows_threaded(probes, gallery, threads)
    rev = knn2_rows_threaded(gallery, probes, threads)[:, 0] if cross_check else None
    rows = []
    for p_i in range(len(probes)):
        idx, best, second = (int(v) for v in fwd[p_i])
        if ratio is not None and not (best < ratio * second):
            continue
        if max_distance is not None and best > max_distance:
            continue
        if rev is not None and rev[idx] != p_i:
            continue
        rows.append((p_i, idx, best, second))
    return np.array(rows, np.int32).reshape(-1, 4)
