"""At-size parity for BASELINE.json configs 3, 4 and 5 (SURVEY.md §8a sizes), through the sharded
drivers a multi-GPU job uses (paper_1609_03986_b200/sharded.py; world of one on this box) and the
C ABI underneath. The CPU side is the oracle restatement on all host threads and, when oracle/_ref
is present, the unmodified reference itself.

  cfg3  two FULL 3840x2160 images x 50 000 keypoints: every descriptor compared
        (reference paths: proj/src/descriptor.cpp:90-105)
        + one frame of non-integer float64 pixels at that size (the float-texture route of the default kernel)
  cfg4  the FULL 1 M x 1 M match: 4 096 sampled rows against the oracle's knn2, every planted copy,
        every duplicated train row (lowest index wins), the ratio pass on all 1 M triples
        (proj/src/match.cpp:33-81)
  cfg5  eight FULL image pairs (8 000 x 8 000, ratio 0.8 + cross-check) from descriptors extracted
        here, against match_brute_force (proj/src/match.cpp:52-81)
"""
import numpy as np
import pytest

import oracle
from oracle import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lk():
    import paper_1609_03986_b200 as pkg
    pkg.get_engine()          # fails loudly here if libclatch.so or the GPU is missing
    return pkg


def test_cfg3_two_full_images(lk):
    from paper_1609_03986_b200 import sharded
    imgs, kps = W.images_and_keypoints("cfg3", [0, 63])
    kps[1][::997, 0] = 20.0                                  # margin violators in one of the images
    got = sharded.extract_images_sharded(imgs, kps)          # -> describe_batch (u8 images)
    assert sorted(got) == [0, 1]
    got64 = lk.describe_batch([imgs[1].astype(np.float64)], [kps[1]])[0]      # reference dtype, banded upload
    ref = oracle.ref()
    for i in (0, 1):
        kept_idx, want = W.describe_all_threaded(imgs[i], kps[i])
        kept, desc = got[i]
        assert desc.shape == (len(want), 64) and len(want) >= 49_900
        assert np.array_equal(kept, kps[i][kept_idx])        # input order, violators dropped
        assert np.array_equal(desc, want), f"cfg3 image {i}: {(desc != want).any(1).sum()} descriptors differ"
    assert np.array_equal(got64[1], got[1][1])
    if ref is not None:                                      # the reference itself on a slice of each image
        for i in (0, 1):
            _, rdesc = ref.describe_all(imgs[i].astype(np.float64), kps[i][:4000], workers=0)
            assert np.array_equal(got[i][1][:len(rdesc)], rdesc)


def test_cfg3_size_frame_of_non_integer_doubles(lk):
    """The float-texture route of the default kernel at cfg3 size: one 3840x2160 frame of float64 pixels that are not
    u8 values (a warped, noisy frame; ordinary numpy memory and page-locked) x 50 000 keypoints, every descriptor
    against the oracle on all host threads (reference path: proj/src/descriptor.cpp:29-105)."""
    torch = pytest.importorskip("torch")
    imgs, kps = W.images_and_keypoints("cfg3", [7])
    rng = np.random.default_rng(1609_7)
    frame = imgs[0].astype(np.float64) * 0.87 + rng.random(imgs[0].shape) * 7.5 - 3.0
    kept_idx, want = W.describe_all_threaded(frame, kps[0])
    assert len(want) >= 49_900
    kept, desc = lk.describe(frame, kps[0])
    assert np.array_equal(kept, kps[0][kept_idx])
    assert np.array_equal(desc, want), f"{(desc != want).any(1).sum()} descriptors differ"
    pin = torch.empty(frame.shape, dtype=torch.float64, pin_memory=True)
    pin.numpy()[...] = frame
    assert np.array_equal(lk.describe(pin.numpy(), kps[0])[1], want)
    assert np.array_equal(lk.describe(frame, kps[0])[1], want)          # (second call from numpy memory: chunked staging)


def test_cfg4_full_match(lk):
    from paper_1609_03986_b200 import sharded
    q, t, (dup_q, src_t) = W.cfg4_sets()
    n = len(q)
    assert n == 1_000_000 and len(t) == n
    eng = lk.get_engine()
    bi, bd, sd = eng.match_top2(q, t)
    trip = np.stack([bi, bd, sd], 1)
    # 4 096 sampled rows (planted copies among them) against the oracle, all host threads
    rng = np.random.default_rng(44)
    rows = np.unique(np.r_[dup_q[:512], rng.integers(0, n, 3584)])
    want = W.knn2_rows_threaded(q[rows], t)
    assert np.array_equal(trip[rows], want), f"{(trip[rows] != want).any(1).sum()} of {len(rows)} sampled rows differ"
    ref = oracle.ref()
    if ref is not None:
        assert np.array_equal(trip[rows[:64]], ref.knn2_all(q[rows[:64]], t))
    # every planted copy is found at distance 0, and at the LOWEST train index holding those bytes
    assert np.all(bd[dup_q] == 0)
    assert np.all(bi[dup_q] <= src_t)
    assert np.array_equal(t[bi[dup_q]], q[dup_q])
    moved = dup_q[bi[dup_q] != src_t]                        # copies of duplicated train rows: tie -> lower index
    assert np.all(sd[moved] == 0)
    # unplanted rows: Binomial(512, 1/2) minimum over 1e6 draws
    mask = np.ones(n, bool); mask[dup_q] = False
    assert bd[mask].min() > 120 and bd[mask].max() < 256 and np.all(sd[mask] >= bd[mask])
    assert np.all((bi >= 0) & (bi < n))
    # the same job from host arrays through the sharded driver, ratio test 0.8 on all 1 M triples
    got = sharded.match_sharded_host(q, t, ratio=W.RATIO)
    keep = bd < W.RATIO * sd                                 # src/match.cpp:70-72 (double arithmetic)
    want_rows = np.stack([np.arange(n, dtype=np.int32)[keep], bi[keep], bd[keep], sd[keep]], 1)
    assert np.array_equal(got, want_rows)
    assert set(dup_q[sd[dup_q] > 0]).issubset(set(got[:, 0]))    # a unique exact copy always passes the ratio test


def test_cfg5_eight_full_pairs(lk):
    from paper_1609_03986_b200 import sharded
    idx = [0, 1, 2, 3, 255]
    imgs, kps = W.images_and_keypoints("cfg5", idx)
    local = sharded.extract_images_sharded(imgs, kps)
    sets = [local[i][1] for i in range(len(idx))]
    for i in (0, 4):
        assert np.array_equal(sets[i], W.describe_all_threaded(imgs[i], kps[i])[1])
    # plant cross-image structure: noise images never match each other, so copy rows (with a few bit
    # flips) from set 0 into the others and duplicate a row inside a set (ties on both passes)
    rng = np.random.default_rng(55)
    sets = [s.copy() for s in sets]
    for j in range(1, len(sets)):
        rows = rng.choice(len(sets[j]), 600, replace=False)
        src = rng.choice(len(sets[0]), 600, replace=False)
        sets[j][rows] = sets[0][src]
        flips = rng.integers(0, 512, (600, 6))
        for r, f in zip(rows[:400], flips):
            for b in f:
                sets[j][r, b >> 3] ^= np.uint8(1 << (b & 7))
        sets[j][rows[-1]] = sets[j][rows[-2]]
    import torch
    dsets = sharded.all_gather_descriptor_sets(dict(enumerate(sets)), len(sets), device=torch.device("cuda", 0))
    got = sharded.match_all_pairs_resident(dsets, ratio=W.RATIO, cross_check=True)
    pairs = sorted(got)
    assert len(pairs) == 10
    ref = oracle.ref()
    total = 0
    for p in pairs[:8]:
        want = W.match_threaded(sets[p[0]], sets[p[1]], ratio=W.RATIO, cross_check=True)
        assert np.array_equal(got[p], want), f"pair {p}: {len(got[p])} rows vs {len(want)}"
        total += len(want)
    assert total > 1000                                      # the filter passes real matches, not an empty set
    if ref is not None:
        p = pairs[0]
        assert np.array_equal(got[p], ref.match(sets[p[0]], sets[p[1]], ratio=W.RATIO, cross_check=True, workers=0))
    # the reference-facing single-pair call gives the same rows
    p = pairs[3]
    assert np.array_equal(lk.match(sets[p[0]], sets[p[1]], ratio=W.RATIO, cross_check=True), got[p])


def test_cuda_against_the_reference_build_directly(lk):
    """The GPU path against oracle/_ref (the unmodified reference compiled from /root/reference), not the
    restatement: describe_all on a structured image and match_brute_force with every filter."""
    ref = oracle.ref()
    if ref is None:
        pytest.skip("oracle/_ref/liblatch_ref.so not built")
    port = oracle.port()
    img = port.structured_image(2024, 800, 600)
    kps = port.random_keypoints(515, 800, 600, 3000)
    kps[::50, 1] = 590.0
    rk, rdesc = ref.describe_all(img, kps, workers=0)
    kept, desc = lk.describe(img, kps)
    assert np.array_equal(desc, rdesc) and np.array_equal(kept, kps[rk])
    assert np.array_equal(lk.describe(img.astype(np.uint8), kps)[1], rdesc)
    g = rdesc.copy()
    g[100] = g[7]
    for kw in ({}, {"ratio": 0.8}, {"cross_check": True}, {"max_distance": 150},
               {"ratio": 0.9, "cross_check": True, "max_distance": 200}):
        assert np.array_equal(lk.match(rdesc, g, **kw), ref.match(rdesc, g, workers=0, **kw)), kw
