"""Pins the CPU checkers (oracle/) before anything trusts them.

The C restatement (oracle/latch_oracle.c) must reproduce (a) the reference's own
golden fixtures and (b) the seeded vectors generated from the unmodified
reference by oracle/make_golden.py; where oracle/_ref is present it is also
compared with the reference live.
"""
import hashlib

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, parse_ltch

SHA = {
    "golden_image.pgm": "fa0ff57b05c3819704cb1f9fe36cc7e19fd708c4fc7ec71879a54b1684054b46",
    "golden_descriptors.bin": "2e5a96aa25d448f9827146424c7fcaa3761c32e480b5934aeb1adb5b4cd8b19a",
    "golden_bits.bin": "a2dcdbd89fa70a08abfaae09d5d6cf82a07a627b9966a90c75609baab6cc5004",
}


def test_fixture_hashes():
    for name, sha in SHA.items():
        assert hashlib.sha256((GOLDEN / name).read_bytes()).hexdigest() == sha


def test_rng_stream(port, vectors):
    assert np.array_equal(port.rng_next(7, 700), vectors["rng_next_7"])
    assert np.array_equal(port.rng_units(7, 16), vectors["rng_units_7"])


def test_golden_bits(port, golden_image_u8):
    # acceptance.cpp:96-118 — keypoint (128,128,0.3), default pattern
    got = port.describe(golden_image_u8.astype(np.float64), [128.0, 128.0, 0.3, 0.0])
    assert got.tobytes() == (GOLDEN / "golden_bits.bin").read_bytes()


def test_golden_descriptor_file(port, golden_image_u8):
    # acceptance.cpp:120-130 — describe_all over the detected keypoints
    kps = np.load(GOLDEN / "golden_keypoints_f64.npy")
    assert kps.shape == (257, 4)
    kept, desc = port.describe_all(golden_image_u8.astype(np.float64), kps)
    fkps, fdesc = parse_ltch((GOLDEN / "golden_descriptors.bin").read_bytes())
    assert len(kept) == len(fdesc) == 257
    assert np.array_equal(desc, fdesc)
    assert np.array_equal(kps[kept].astype(np.float32), fkps)


def test_windows(port, vectors):
    seed, w, h = (int(v) for v in vectors["win_image_seed"])
    img = port.structured_image(seed, w, h)
    for kp, want in zip(vectors["win_kps"], vectors["win_values"]):
        assert np.array_equal(port.extract_window(img, kp), want)  # exact == on doubles


@pytest.mark.parametrize("tag,maker,args", [("struct", "structured_image", (83, 160, 160)),
                                            ("noise", "random_image", (1609, 200, 150))])
def test_describe_all_vectors(port, vectors, tag, maker, args):
    img = getattr(port, maker)(*args)
    kept, desc = port.describe_all(img, vectors[f"desc_{tag}_kps"])
    assert np.array_equal(kept, vectors[f"desc_{tag}_kept"])
    assert np.array_equal(desc, vectors[f"desc_{tag}_out"])
    assert 4 not in kept and 5 not in kept  # the planted margin violators


@pytest.mark.parametrize("name", ["t8k8", "t64k5w", "t16k12z", "t24k1"])
def test_custom_patterns(port, vectors, name):
    img = port.structured_image(97, 140, 140)
    pat = oracle.parse_pattern_text((GOLDEN / f"pattern_{name}.latchpat").read_text())
    kept, desc = port.describe_all(img, vectors["pat_kps"], pattern=pat)
    assert np.array_equal(desc, vectors[f"pat_{name}_out"])


def _planted(port, seed, q, n, nbytes=64):
    d = port.random_descriptors(seed, q + n, nbytes)
    return d[:q].copy(), d[q:].copy()


def test_match_vectors_131(port, vectors):
    probes, gallery = _planted(port, 131, 60, 45)
    gallery[10] = gallery[3]
    gallery[44] = gallery[7]
    probes[5] = gallery[3]
    assert np.array_equal(port.knn2_all(probes, gallery), vectors["m131_knn2"])
    for combo in range(8):
        got = port.match(probes, gallery, ratio=0.9 if combo & 1 else None,
                         cross_check=bool(combo & 2), max_distance=250 if combo & 4 else None)
        assert np.array_equal(got, vectors[f"m131_combo{combo}"])


def test_match_vectors_515(port, vectors):
    probes, gallery = _planted(port, 515, 500, 500)
    gallery[7] = gallery[3]
    gallery[450] = gallery[11]
    probes[5] = gallery[3]
    probes[301] = probes[5]
    assert np.array_equal(port.knn2_all(probes, gallery), vectors["m515_knn2"])
    for combo in range(8):
        got = port.match(probes, gallery, ratio=0.8 if combo & 1 else None,
                         cross_check=bool(combo & 2), max_distance=240 if combo & 4 else None)
        assert np.array_equal(got, vectors[f"m515_combo{combo}"])


def test_tail_bytes(port, vectors):
    probes, gallery = _planted(port, 113, 20, 33, 13)
    assert np.array_equal(port.knn2_all(probes, gallery), vectors["m113_knn2"])
    a, b = probes[0], gallery[0]
    assert port.hamming(a, b) == int(np.unpackbits(a ^ b).sum())


def test_known_answers(port):
    # test_match.cpp:41-47, 68-81
    def ones(k):
        bits = np.zeros(512, np.uint8)
        bits[:k] = 1
        return np.packbits(bits, bitorder="little")
    assert port.hamming(ones(512), ones(0)) == 512
    assert port.hamming(ones(200), ones(137)) == 63
    gallery = np.stack([ones(10), ones(3), ones(7), ones(3)])
    assert port.knn2(ones(0), gallery) == (1, 3, 3)
    assert port.knn2(ones(0), np.stack([ones(9)])) == (0, 9, 513)
    with pytest.raises(RuntimeError):
        port.match(np.stack([ones(1)]), np.zeros((0, 64), np.uint8))
    assert len(port.match(np.zeros((0, 64), np.uint8), np.stack([ones(1)]))) == 0
    # margin: test_descriptor.cpp:76-87
    assert port.in_margin(93, 93, 46.0, 46.0)
    assert not port.in_margin(93, 93, 45.999, 46.0)
    assert port.in_margin(200, 100, 153.0, 53.0)
    assert not port.in_margin(200, 100, 154.0, 53.0)
    assert not port.in_margin(200, 100, float("nan"), 53.0)


# ---- live comparison with the unmodified reference (when oracle/_ref exists) ----

def test_pattern_file_is_reference_default(ref):
    T, K, trip, weights = ref.parse_pattern(ref.default_pattern_text())
    t2, k2, trip2, w2 = oracle.default_pattern()
    assert (T, K) == (t2, k2) and np.array_equal(trip, trip2) and np.array_equal(weights, w2)
    from paper_1609_03986_b200.pattern import default_pattern_text
    assert default_pattern_text() == ref.default_pattern_text()


def test_port_equals_reference_live(port, ref):
    assert np.array_equal(port.random_image(5, 97, 61), ref.random_image(5, 97, 61))
    assert np.array_equal(port.structured_image(9, 150, 120), ref.structured_image(9, 150, 120))
    assert np.array_equal(port.random_descriptors(3, 50, 64), ref.random_descriptors(3, 50, 64))
    assert np.array_equal(port.random_image_u8(5, 97, 61).astype(np.float64),
                          ref.random_image(5, 97, 61))
    img = ref.structured_image(2024, 256, 192)
    kps = port.random_keypoints(77, 256, 192, 300)
    kps[::50, 0] = 3.0  # margin violators
    k1, d1 = port.describe_all(img, kps)
    k2, d2 = ref.describe_all(img, kps)
    assert np.array_equal(k1, k2) and np.array_equal(d1, d2)
    # non-integer image (eval.cpp:76-84 produces these)
    rng = np.random.default_rng(0)
    fimg = rng.random((150, 170)) * 255.0
    kps = port.random_keypoints(78, 170, 150, 100)
    assert np.array_equal(port.describe_all(fimg, kps)[1], ref.describe_all(fimg, kps)[1])
    probes, gallery = ref.random_descriptors(41, 300, 64), ref.random_descriptors(42, 400, 64)
    gallery[17] = gallery[250]
    probes[3] = gallery[250]
    assert np.array_equal(port.knn2_all(probes, gallery), ref.knn2_all(probes, gallery))
    for kw in ({}, {"ratio": 0.8}, {"cross_check": True}, {"max_distance": 230},
               {"ratio": 0.85, "cross_check": True, "max_distance": 235}):
        assert np.array_equal(port.match(probes, gallery, **kw), ref.match(probes, gallery, **kw))


# ---- detection (next row): restatement vs golden keypoints, vectors and the live reference ----

DET_CASES = [("struct", "structured_image", (1, 160, 120), 20.0, True, True),
             ("noise", "random_image", (2, 96, 80), 30.5, True, True),
             ("nonms", "random_image", (3, 64, 48), 12.25, False, False)]


def test_detect_golden_keypoints(port, golden_image_u8):
    want = np.load(GOLDEN / "golden_keypoints_f64.npy")
    assert np.array_equal(port.detect(golden_image_u8.astype(np.float64), 20.0, True, True), want)


@pytest.mark.parametrize("tag,maker,args,thr,nms,ori", DET_CASES)
def test_detect_vectors(port, vectors, tag, maker, args, thr, nms, ori):
    got = port.detect(getattr(port, maker)(*args), thr, nms, ori)
    assert np.array_equal(got, vectors[f"det_{tag}_out"])


def test_detect_non_integer_image(port, vectors):
    assert np.array_equal(port.detect(vectors["det_frac_image"], 40.0, True, True), vectors["det_frac_out"])


def test_detect_live_reference(port, ref):
    for seed, (w, h), thr, nms, ori in [(5, (320, 240), 20.0, True, True), (6, (200, 150), 25.5, False, True),
                                        (7, (97, 61), 20.0, True, False)]:
        for maker in ("structured_image", "random_image"):
            im = getattr(port, maker)(seed, w, h)
            assert np.array_equal(port.detect(im, thr, nms, ori), ref.detect(im, thr, nms, ori))
    with pytest.raises(RuntimeError):
        port.detect(np.zeros((32, 6)))


# ---- trainer scoring (next row): candidate bits over upright patches ----

def _score_windows(port):
    wins = np.stack([port.random_image(300 + i, 64, 64) for i in range(45)])
    wins[40:] = np.stack([port.structured_image(400 + i, 64, 64) for i in range(5)])
    return wins


def test_triplet_bits_vectors(port, vectors):
    wins = _score_windows(port)
    _, _, _, seven = oracle.default_pattern()
    assert np.array_equal(port.triplet_bits(wins, vectors["score_candidates_k8"], 8, seven), vectors["score_bits_seven"])
    assert np.array_equal(port.triplet_bits(wins, vectors["score_candidates_k8"], 8, np.ones(64)),
                          vectors["score_bits_ones"])
    assert np.array_equal(port.triplet_bits(wins, vectors["score_candidates_k5"], 5, vectors["score_weights_k5"]),
                          vectors["score_bits_k5"])
