"""Parity tests proper: the CUDA path, called through the C ABI (ctypes -> libclatch.so),
against the reference's golden fixtures, the committed reference vectors and the CPU
oracle on the same seeded inputs. Bit-exact everywhere (bytes, indices, distances).

Test names follow the reference's own suites (proj/tests/test_descriptor.cpp,
test_match.cpp, acceptance.cpp, python/test_smoke.py).
"""
import numpy as np
import pytest

import oracle
from conftest import GOLDEN, parse_ltch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lk():
    import paper_1609_03986_b200 as pkg
    pkg.get_engine()          # fails loudly here if libclatch.so or the GPU is missing
    return pkg


# ---------------------------------------------------------------- extraction ----

def test_golden_bits(lk, golden_image_u8):
    # acceptance.cpp:96-118
    want = (GOLDEN / "golden_bits.bin").read_bytes()
    for img in (golden_image_u8, golden_image_u8.astype(np.float64)):
        kept, desc = lk.describe(img, np.array([[128.0, 128.0, 0.3, 0.0]]))
        assert desc.shape == (1, 64) and desc.dtype == np.uint8
        assert desc[0].tobytes() == want


def test_golden_descriptor_file(lk, golden_image_u8):
    # acceptance.cpp:120-130
    kps = np.load(GOLDEN / "golden_keypoints_f64.npy")
    blob = (GOLDEN / "golden_descriptors.bin").read_bytes()
    fkps, fdesc = parse_ltch(blob)
    for img in (golden_image_u8, golden_image_u8.astype(np.float64)):
        kept, desc = lk.describe(img, kps)
        assert np.array_equal(desc, fdesc)
        assert np.array_equal(kept.astype(np.float32), fkps)
        assert lk.format_descriptor_file(kept, desc) == blob            # the LTCH file, byte for byte
    # detect -> describe -> file, the reference's `latch describe` pipeline end to end
    kept, desc = lk.describe(golden_image_u8, lk.detect(golden_image_u8))
    assert lk.format_descriptor_file(kept, desc) == blob


@pytest.mark.parametrize("tag,maker,args", [("struct", "structured_image", (83, 160, 160)),
                                            ("noise", "random_image", (1609, 200, 150))])
def test_reference_vectors(lk, port, vectors, tag, maker, args):
    img = getattr(port, maker)(*args)
    kps = vectors[f"desc_{tag}_kps"]
    for im in (img, img.astype(np.uint8)):
        kept, desc = lk.describe(im, kps)
        assert np.array_equal(kept, kps[vectors[f"desc_{tag}_kept"]])   # order kept, violators dropped
        assert np.array_equal(desc, vectors[f"desc_{tag}_out"])


@pytest.mark.parametrize("name", ["t8k8", "t64k5w", "t16k12z", "t24k1"])
def test_custom_patterns(lk, port, vectors, name):
    # generic kernel: python/test_smoke.py:105-123 describes with a T=8 pattern
    img = port.structured_image(97, 140, 140)
    text = (GOLDEN / f"pattern_{name}.latchpat").read_text()
    for im in (img, img.astype(np.uint8)):
        kept, desc = lk.describe(im, vectors["pat_kps"], pattern=text)
        assert desc.shape == vectors[f"pat_{name}_out"].shape
        assert np.array_equal(desc, vectors[f"pat_{name}_out"])
    # and back to the built-in pattern on the same context
    kept, desc = lk.describe(img, vectors["pat_kps"][:4])
    assert np.array_equal(desc, port.describe_all(img, vectors["pat_kps"][:4])[1])


def test_default_pattern_text_matches_builtin(lk, port):
    # python/test_smoke.py:96-103
    text = lk.default_pattern()
    assert text.startswith("LATCHPAT v1 T=512 K=8\n")
    img = port.structured_image(5, 150, 150)
    kps = port.random_keypoints(6, 150, 150, 40)
    _, implicit = lk.describe(img, kps)
    _, explicit = lk.describe(img, kps, pattern=text)
    assert np.array_equal(implicit, explicit)


def test_describe_all_drops_margin_violators(lk, port):
    # test_descriptor.cpp:178-201
    img = port.structured_image(101, 140, 140)
    kps = np.array([[50.0, 50.0, 0.5, 9.0], [10.0, 70.0, 0.0, 8.0], [70.0, 50.0, -0.5, 7.0],
                    [70.0, 139.0, 0.0, 6.0], [93.0, 93.0, 2.0, 5.0]])
    kept, desc = lk.describe(img, kps, workers=1)
    assert len(kept) == 3
    assert np.array_equal(kept, kps[[0, 2, 4]])            # theta and score pass through
    for k, d in zip(kept, desc):
        assert np.array_equal(d, port.describe(img, k))
    for workers in (2, 8):
        assert np.array_equal(lk.describe(img, kps, workers=workers)[1], desc)
    # bare (x, y) rows get theta = 0 (python/test_smoke.py:49-52)
    upright, d0 = lk.describe(img, kps[:, :2])
    assert upright.shape == (3, 4) and np.all(upright[:, 2:] == 0.0)
    assert np.array_equal(d0[0], port.describe(img, [50.0, 50.0, 0.0, 0.0]))
    # nothing inside the margin
    kept, desc = lk.describe(img, np.array([[1.0, 1.0, 0.0, 0.0]]))
    assert kept.shape == (0, 4) and desc.shape == (0, 64)
    kept, desc = lk.describe(img, np.zeros((0, 4)))
    assert kept.shape == (0, 4) and desc.shape == (0, 64)


def test_margin_edges_and_special_angles(lk, port):
    # test_descriptor.cpp:57-87: half-integer centre, half turn, exact 46 px margin
    img = port.random_image(67, 128, 128)
    kps = np.array([[63.5, 63.5, 0.0, 0.0], [63.5, 63.5, np.pi, 0.0], [46.0, 46.0, 1.0, 0.0],
                    [81.0, 81.0, -2.0, 0.0], [46.0, 81.0, np.pi / 2, 0.0],
                    [45.999, 46.0, 0.0, 0.0], [46.0, 81.001, 0.0, 0.0], [np.nan, 60.0, 0.0, 0.0]])
    kept, desc = lk.describe(img, kps)
    want_kept, want = port.describe_all(img, kps)
    assert list(want_kept) == [0, 1, 2, 3, 4]
    assert np.array_equal(kept, kps[want_kept]) and np.array_equal(desc, want)


def test_brightness_invariance(lk, port):
    # test_descriptor.cpp:145-161, acceptance.cpp:260-280 (exact)
    img = port.structured_image(89, 128, 128)
    kps = port.random_keypoints(90, 128, 128, 30)
    _, base = lk.describe(img, kps)
    for shift in (30.0, -50.0, 1.0):
        _, d = lk.describe(img + shift, kps)
        assert np.array_equal(d, base)


def test_non_integer_image_uses_f64_sampling(lk, port):
    # eval.cpp:76-84 produces non-integer images (warp + noise): no u8 promotion possible
    rng = np.random.default_rng(0)
    img = rng.random((150, 170)) * 255.0
    kps = port.random_keypoints(78, 170, 150, 120)
    kept, desc = lk.describe(img, kps)
    assert np.array_equal(desc, port.describe_all(img, kps)[1])
    # one fractional pixel far from every window must still disable promotion safely
    img2 = port.structured_image(3, 170, 150)
    img2[0, 0] = 0.5
    assert np.array_equal(lk.describe(img2, kps)[1], port.describe_all(img2, kps)[1])
    # float32 input is force-cast like the reference does
    img3 = port.random_image(4, 170, 150).astype(np.float32)
    assert np.array_equal(lk.describe(img3, kps)[1], port.describe_all(img3.astype(np.float64), kps)[1])


def test_strided_and_odd_width_images(lk, port):
    # pitch not a multiple of 16 and non-contiguous rows exercise the staging paths
    full = port.random_image_u8(12, 333, 201)
    kps = port.random_keypoints(13, 301, 190, 80)
    view = full[5:195, 16:317]                 # 190 x 301 window into a wider buffer
    want = port.describe_all(np.ascontiguousarray(view).astype(np.float64), kps)[1]
    assert np.array_equal(lk.describe(view, kps)[1], want)
    assert np.array_equal(lk.describe(np.ascontiguousarray(view), kps)[1], want)
    assert np.array_equal(lk.describe(view.astype(np.float64), kps)[1], want)


@pytest.mark.parametrize("w,h,n,img_seed,kp_seed", [(640, 480, 2000, 1609, 1610),     # BASELINE cfg1
                                                    (1920, 1080, 10000, 3986, 3987)])  # BASELINE cfg2
def test_baseline_configs_extract_and_match(lk, port, w, h, n, img_seed, kp_seed):
    img_u8 = port.random_image_u8(img_seed, w, h)
    kps = port.random_keypoints(kp_seed, w, h, n)
    kps[::97, 1] = 20.0                        # ~1 % margin violators
    kept, desc = lk.describe(img_u8, kps)
    want_kept, want = port.describe_all(img_u8.astype(np.float64), kps)
    assert np.array_equal(kept, kps[want_kept])
    assert np.array_equal(desc, want)
    # top-2 self-match with planted duplicates (ties -> lowest index)
    gallery = desc.copy()
    gallery[len(gallery) // 2] = gallery[11]
    gallery[-1] = gallery[12]
    eng = lk.get_engine()
    bi, bd, sd = eng.match_top2(desc, gallery)
    # oracle on a sample of rows at cfg2 size, all rows at cfg1 size
    rows = np.arange(len(desc)) if n <= 2000 else np.unique(
        np.r_[0:64, 11, 12, len(desc) // 2, len(desc) - 1, np.random.default_rng(1).integers(0, len(desc), 400)])
    want3 = port.knn2_all(desc[rows], gallery)
    assert np.array_equal(np.stack([bi, bd, sd], 1)[rows], want3)
    assert bi[11] == 11 and bd[11] == 0 and sd[11] == 0        # duplicate is the runner-up
    assert bi[12] == 12 and sd[12] == 0                        # lowest index wins the tie


def test_structured_large_image(lk, port):
    # flat regions make d1 ~ d2 ~ rounding noise: the hardest case for bit parity
    img = port.structured_image(2024, 800, 600)
    kps = port.random_keypoints(2025, 800, 600, 1500)
    assert np.array_equal(lk.describe(img, kps)[1], port.describe_all(img, kps)[1])


def test_extract_device_api(lk, port):
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_pattern(None)
    img = port.random_image_u8(7, 640, 480)
    kps = port.random_keypoints(8, 640, 480, 500)
    xycs, kept = eng.prepare_keypoints(kps, 640, 480)
    want = port.describe_all(img.astype(np.float64), kps)[1]
    d_xycs = torch.from_numpy(xycs).cuda()
    for host_img in (img, img.astype(np.float64)):
        out = eng.extract_device(torch.from_numpy(host_img).cuda(), d_xycs)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)
    # side stream
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        out = eng.extract_device(torch.from_numpy(img).cuda(), d_xycs)
    st.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)


# ------------------------------------------------------------------ matching ----

def _ones(k, nbytes=64):
    bits = np.zeros(nbytes * 8, np.uint8)
    bits[:k] = 1
    return np.packbits(bits, bitorder="little")


def test_hamming_counts_differing_bits(lk, port):
    # test_match.cpp:41-66
    assert lk.hamming(np.array([0x00], np.uint8), np.array([0x00], np.uint8)) == 0
    assert lk.hamming(np.array([0xff], np.uint8), np.array([0x00], np.uint8)) == 8
    assert lk.hamming(np.array([0xaa], np.uint8), np.array([0x55], np.uint8)) == 8
    assert lk.hamming(np.array([0x0f, 0xf0], np.uint8), np.array([0x00, 0xf0], np.uint8)) == 4
    assert lk.hamming(_ones(512), _ones(0)) == 512
    assert lk.hamming(_ones(200), _ones(137)) == 63
    with pytest.raises(RuntimeError):
        lk.hamming(np.zeros(1, np.uint8), np.zeros(2, np.uint8))
    d = port.random_descriptors(109, 40, 64)
    for a, b in zip(d[::2], d[1::2]):
        assert lk.hamming(a, b) == port.hamming(a, b) == lk.hamming(b, a)
        assert lk.hamming(a, a) == 0
    t = port.random_descriptors(113, 20, 13)       # byte tail
    for a, b in zip(t[::2], t[1::2]):
        assert lk.hamming(a, b) == int(np.unpackbits(a ^ b).sum())


def test_knn2_ties_and_sentinel(lk):
    # test_match.cpp:68-81
    eng = lk.get_engine()
    gallery = np.stack([_ones(10), _ones(3), _ones(7), _ones(3)])
    bi, bd, sd = eng.match_top2(_ones(0)[None], gallery)
    assert (bi[0], bd[0], sd[0]) == (1, 3, 3)
    bi, bd, sd = eng.match_top2(_ones(0)[None], _ones(9)[None])
    assert (bi[0], bd[0], sd[0]) == (0, 9, 513)


def test_filters_known_answers(lk):
    # test_match.cpp:105-158
    p0 = _ones(0)[None]
    assert len(lk.match(p0, np.stack([_ones(4), _ones(4)]), ratio=1.0)) == 0      # strict <
    spread = np.stack([_ones(4), _ones(9)])
    kept = lk.match(p0, spread, ratio=0.5)
    assert kept.tolist() == [[0, 0, 4, 9]]
    assert len(lk.match(p0, spread, ratio=0.4)) == 0
    assert len(lk.match(p0, _ones(400)[None], ratio=0.8)) == 1                    # sentinel 513
    assert len(lk.match(p0, _ones(7)[None], max_distance=7)) == 1                 # inclusive
    assert len(lk.match(p0, _ones(7)[None], max_distance=6)) == 0
    probes = np.stack([_ones(1), _ones(2)])
    gallery = np.stack([_ones(0), _ones(30)])
    got = lk.match(probes, gallery, cross_check=True)
    assert got.tolist() == [[0, 0, 1, 29]]
    assert len(lk.match(probes, gallery)) == 2


@pytest.mark.parametrize("seed,q,n,ratio,maxd", [(131, 60, 45, 0.9, 250), (515, 500, 500, 0.8, 240)])
def test_matcher_every_filter_combination(lk, port, vectors, seed, q, n, ratio, maxd):
    # test_match.cpp:160-188 and acceptance.cpp:164-216
    d = port.random_descriptors(seed, q + n, 64)
    probes, gallery = d[:q].copy(), d[q:].copy()
    if seed == 131:
        gallery[10] = gallery[3]; gallery[44] = gallery[7]; probes[5] = gallery[3]
    else:
        gallery[7] = gallery[3]; gallery[450] = gallery[11]; probes[5] = gallery[3]; probes[301] = probes[5]
    bi, bd, sd = lk.get_engine().match_top2(probes, gallery)
    assert np.array_equal(np.stack([bi, bd, sd], 1), vectors[f"m{seed}_knn2"])
    for combo in range(8):
        kw = dict(ratio=ratio if combo & 1 else None, cross_check=bool(combo & 2),
                  max_distance=maxd if combo & 4 else None)
        want = vectors[f"m{seed}_combo{combo}"]
        for workers in (1, 2, 8):
            got = lk.match(probes, gallery, workers=workers, **kw)
            assert got.dtype == np.int32 and np.array_equal(got, want)
        assert np.all(np.diff(got[:, 0]) > 0)


def test_tail_length_descriptors(lk, port, vectors):
    d = port.random_descriptors(113, 53, 13)
    probes, gallery = d[:20].copy(), d[20:].copy()
    bi, bd, sd = lk.get_engine().match_top2(probes, gallery)
    assert np.array_equal(np.stack([bi, bd, sd], 1), vectors["m113_knn2"])
    for nbytes in (1, 8, 32, 100):
        dd = port.random_descriptors(nbytes, 70, nbytes)
        assert np.array_equal(lk.match(dd[:30], dd[30:], ratio=0.95),
                              port.match(dd[:30], dd[30:], ratio=0.95))


def test_match_edge_cases(lk):
    # test_match.cpp:190-192, python/test_smoke.py:126-136
    with pytest.raises(RuntimeError):
        lk.match(np.zeros((2, 64), np.uint8), np.zeros((0, 64), np.uint8))
    with pytest.raises(RuntimeError):
        lk.match(np.zeros((0, 64), np.uint8), np.zeros((0, 64), np.uint8))   # gallery checked first
    empty = lk.match(np.zeros((0, 64), np.uint8), np.zeros((3, 64), np.uint8))
    assert empty.shape == (0, 4) and empty.dtype == np.int32
    with pytest.raises(ValueError):
        lk.match(np.zeros(64, np.uint8), np.zeros((3, 64), np.uint8))
    with pytest.raises(RuntimeError):
        lk.match(np.zeros((2, 64), np.uint8), np.zeros((3, 32), np.uint8))


@pytest.mark.parametrize("q,n", [(1, 1), (1, 127), (3, 128), (130, 129), (257, 1000), (5, 40000),
                                 (1000, 1), (4096, 4097)])
def test_ragged_shapes_against_oracle(lk, port, q, n):
    # tile tails, split tails, more CTAs than work, a single train row
    d = port.random_descriptors(1000 + q + n, q + n, 64)
    probes, gallery = d[:q].copy(), d[q:].copy()
    if n > 3:
        gallery[n - 1] = gallery[0]            # tie between the first and the last split
        probes[0] = gallery[0]
    bi, bd, sd = lk.get_engine().match_top2(probes, gallery)
    assert np.array_equal(np.stack([bi, bd, sd], 1), port.knn2_all(probes, gallery))


def test_self_match_properties_large(lk, port):
    # size-independent properties at 100k x 100k (1e10 compares; no CPU oracle at this size)
    n = 100_000
    d = port.random_descriptors(41, n, 64)
    d[70_000] = d[123]                          # planted duplicate pair
    d[99_999] = d[0]
    bi, bd, sd = lk.get_engine().match_top2(d, d)
    assert np.all(bd == 0)                      # every row finds itself (or an identical row)
    assert np.all(bi <= np.arange(n))           # ... at the lowest such index
    assert bi[70_000] == 123 and sd[70_000] == 0 and sd[123] == 0
    assert bi[99_999] == 0 and sd[0] == 0
    mask = np.ones(n, bool); mask[[0, 123, 70_000, 99_999]] = False
    assert np.all(bi[mask] == np.arange(n)[mask])
    assert np.all((sd[mask] > 150) & (sd[mask] < 256))   # Binomial(512, 1/2) minimum over 1e5 draws
    rows = np.random.default_rng(3).integers(0, n, 48)
    assert np.array_equal(np.stack([bi, bd, sd], 1)[rows], port.knn2_all(d[rows], d))


def test_match_device_api(lk, port):
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    d = port.random_descriptors(9, 3000, 64)
    probes, gallery = d[:1000].copy(), d[1000:].copy()
    out = eng.match_top2_device(torch.from_numpy(probes).cuda(), torch.from_numpy(gallery).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().T, port.knn2_all(probes, gallery))


def test_python_smoke_shapes(lk, golden_image_u8):
    # python/test_smoke.py:30-53 without detect(): the golden keypoints stand in
    golden = golden_image_u8.astype(np.float64)
    keypoints = np.load(GOLDEN / "golden_keypoints_f64.npy")
    kept, desc = lk.describe(golden, keypoints)
    assert desc.dtype == np.uint8 and desc.shape == (len(kept), lk.descriptor_bytes)
    assert 0 < len(kept) <= len(keypoints)
    matches = lk.match(desc, desc)
    assert matches.shape == (len(desc), 4)
    assert np.array_equal(matches[:, 0], np.arange(len(desc)))
    assert np.all(matches[:, 2] == 0)
    assert np.array_equal(desc[matches[:, 1]], desc[matches[:, 0]])
    assert np.array_equal(lk.match(desc, desc, workers=2), matches)
    a, b = desc[0], desc[1]
    assert lk.hamming(a, b) == int(np.unpackbits(a ^ b).sum())
    with pytest.raises(RuntimeError):
        lk.describe(np.zeros((128, 128)), np.array([[64.0, 64.0]]), pattern="not a pattern")
    with pytest.raises(ValueError):
        lk.describe(np.zeros(16), np.array([[64.0, 64.0]]))


# ------------------------------------------------- matcher kernel variants ----

@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_every_matcher_variant_is_exact(lk, port, variant):
    """All five 64-byte matcher kernels (plain popc, two carry-save forms, tcgen05 int8 and FP4 GEMMs)
    must give the reference's knn2 triples bit for bit, including ties, tails and a lone row."""
    eng = lk.get_engine()
    eng.set_option("match_variant", variant)
    eng.set_option("match_form_auto", 0)             # variant 4 means the e2m1 form at every size here
    try:
        for q, n in [(1, 1), (5, 255), (129, 256), (130, 257), (300, 1000), (1000, 5000), (77, 40000), (7000, 7000)]:
            d = port.random_descriptors(7000 + q + n, q + n, 64)
            probes, gallery = d[:q].copy(), d[q:].copy()
            if n > 3:
                gallery[n - 1] = gallery[0]
                gallery[n // 2] = gallery[1]
                probes[0] = gallery[0]
                probes[q - 1] = gallery[1]
            bi, bd, sd = eng.match_top2(probes, gallery)
            assert np.array_equal(np.stack([bi, bd, sd], 1), port.knn2_all(probes, gallery)), (variant, q, n)
        # extremes of the distance range: all-zero vs all-one rows, and exact duplicates
        probes = np.zeros((3, 64), np.uint8)
        probes[1] = 0xFF
        probes[2, :32] = 0xFF
        gallery = np.stack([np.full(64, 0xFF, np.uint8), np.zeros(64, np.uint8), np.zeros(64, np.uint8)])
        bi, bd, sd = eng.match_top2(probes, gallery)
        assert np.array_equal(np.stack([bi, bd, sd], 1), port.knn2_all(probes, gallery))
        assert (bi[0], bd[0], sd[0]) == (1, 0, 0) and (bi[1], bd[1], sd[1]) == (0, 0, 512)
        # every distance above 256 (all dot products negative): the f32 epilogue's full-pass route
        gallery = ~np.repeat(probes[2:3], 300, 0)
        gallery[::7, 0] ^= 1
        gallery[5, 1] ^= 3
        bi, bd, sd = eng.match_top2(probes[2:3], gallery)
        assert np.array_equal(np.stack([bi, bd, sd], 1), port.knn2_all(probes[2:3], gallery)) and bd[0] > 500
    finally:
        eng.set_option("match_variant", 4)
        eng.set_option("match_form_auto", 1)


@pytest.mark.parametrize("shape", [(1, 1), (1, 300), (129, 257), (700, 513), (2000, 2000), (5000, 9000),
                                   (10000, 10000), (300, 70000), (256, 1), (385, 66000), (40000, 3000)])
def test_tensor_matcher_partitions_agree(lk, port, shape):
    """Small problems are cut "stream-K" style (every CTA an equal run of (query tile, train tile)
    units, pieces merged per query tile), larger ones by (query tile, train split) rounds. Both
    partitions must give the oracle's top-2 — planted duplicates put ties on piece boundaries."""
    q_n, t_n = shape
    rng = np.random.default_rng(q_n * 31 + t_n)
    train = port.random_descriptors(700 + t_n, t_n)
    query = port.random_descriptors(900 + q_n, q_n)
    for j in range(0, q_n, 7):                          # exact copies, each present twice or more in train
        src = int(rng.integers(0, t_n))
        query[j] = train[src]
        train[int(rng.integers(0, t_n))] = train[src]
        for edge in (255, 256, 511, 512, 1023, 1024):   # ... and right at train-tile boundaries
            if edge < t_n and rng.random() < 0.3:
                train[edge] = train[src]
    eng = lk.get_engine()
    res = {}
    try:
        for sk in (1, 0):
            eng.set_option("match_streamk", sk)
            res[sk] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_streamk", 1)
        eng.set_option("match_streamk_pairs", 1)        # stream-K runs on CTA pairs (default: single CTAs)
        res[6] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_2cta", 1)                 # ... as one M = 256 MMA stream per pair (tcgen05 cta_group::2)
        res[7] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_streamk", 0)              # ... and the (query tile pair, split) rounds in that form
        res[8] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_streamk", 1)
        eng.set_option("match_2cta", 0)
        eng.set_option("match_streamk_pairs", 0)
        eng.set_option("match_streamk", 0)
        eng.set_option("match_form_auto", 0)            # e2m1 operands at every size
        eng.set_option("match_pairs", 0)                # every CTA streams the train set for itself
        res[2] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_variant", 3)              # int8 operands (default: e2m1)
        res[3] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_pairs", 1)
        res[4] = np.stack(eng.match_top2(query, train))
        eng.set_option("match_streamk", 1)
        res[5] = np.stack(eng.match_top2(query, train))
    finally:
        eng.set_option("match_streamk", 1)
        eng.set_option("match_streamk_pairs", 0)
        eng.set_option("match_2cta", 0)
        eng.set_option("match_pairs", 1)                # default: CTA pairs share the stream by TMA multicast
        eng.set_option("match_variant", 4)
        eng.set_option("match_form_auto", 1)
    for k in (1, 2, 3, 4, 5, 6, 7, 8):
        assert np.array_equal(res[0], res[k]), k
    rows = np.arange(q_n) if q_n * t_n <= 4_000_000 else np.unique(np.r_[np.arange(0, q_n, 7)[:40], rng.integers(0, q_n, 40)])
    assert np.array_equal(res[1][:, rows].T, port.knn2_all(query[rows], train))


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6])
def test_every_extraction_variant_is_exact(lk, port, variant):
    """All specialised extraction kernels (one window per CTA / four fp64 windows per CTA / four
    split windows with the fp32 filter / the producer-consumer pipeline over the texture unit)
    must be bit-identical to the oracle, including keypoint counts that do not fill a quad."""
    eng = lk.get_engine()
    eng.set_option("extract_variant", variant)
    try:
        img = port.structured_image(2030 + variant, 400, 300)
        for n in (1, 2, 3, 5, 127, 1001):
            kps = port.random_keypoints(2040 + n, 400, 300, n)
            want = port.describe_all(img, kps)[1]
            assert np.array_equal(lk.describe(img.astype(np.uint8), kps)[1], want), (variant, n, "u8")
            assert np.array_equal(lk.describe(img, kps)[1], want), (variant, n, "f64")
        fimg = np.random.default_rng(variant).random((300, 400)) * 255.0
        kps = port.random_keypoints(2050, 400, 300, 203)
        assert np.array_equal(lk.describe(fimg, kps)[1], port.describe_all(fimg, kps)[1])
    finally:
        eng.set_option("extract_variant", 5)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6])
def test_trained_pattern_on_every_fast_kernel(lk, port, variant):
    """A trained pattern has the built-in shape (T=512, K=8, 7x7-of-8x8 mask) but other triplets:
    it takes the specialised kernels with a lane placement planned at clatch_set_pattern time
    (the shipped placement only fits the built-in table). Clustered coordinates make the bank
    residues as unbalanced as a real table can be."""
    rng = np.random.default_rng(5120 + variant)
    trip = rng.integers(0, 57, (512, 6))
    trip[:128, :] = rng.integers(0, 8, (128, 6)) * 8            # all residues equal: worst case for the planner
    trip[128:160, 2:4] = trip[128:160, 0:2]                      # companion b on top of the anchor
    same = (trip[:, 2] == trip[:, 4]) & (trip[:, 3] == trip[:, 5])
    trip[same, 4] = (trip[same, 4] + 1) % 57                     # companions must differ (DegenerateTriplet)
    mask = np.ones((8, 8))
    mask[7, :] = 0.0
    mask[:, 7] = 0.0
    text = "LATCHPAT v1 T=512 K=8\n" + "".join(" ".join(map(str, t)) + "\n" for t in trip)
    text += "WEIGHTS\n" + "".join(" ".join("%.17g" % v for v in row) + "\n" for row in mask)
    pat = (512, 8, trip.astype(np.int32), mask.reshape(-1))
    eng = lk.get_engine()
    eng.set_option("extract_variant", variant)
    try:
        for img in (port.random_image_u8(88, 300, 200), port.structured_image(89, 300, 200).astype(np.uint8)):
            kps = port.random_keypoints(90, 300, 200, 333)
            want = port.describe_all(img.astype(np.float64), kps, pattern=pat)[1]
            assert np.array_equal(lk.describe(img, kps, pattern=text)[1], want)
            assert np.array_equal(lk.describe(img.astype(np.float64), kps, pattern=text)[1], want)
    finally:
        eng.set_option("extract_variant", 5)
        lk.describe(port.random_image_u8(88, 300, 200), port.random_keypoints(90, 300, 200, 4))   # built-in table back


@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6])
def test_smallest_images_and_odd_pitches(lk, port, variant):
    """93x93 is the smallest image with a describable keypoint (46, 46); widths that are not
    multiples of 16 take the unaligned staging / array-fill paths when the image arrives as a
    device tensor with pitch == width."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_option("extract_variant", variant)
    try:
        for w, h in ((93, 93), (94, 93), (107, 131), (160, 97)):
            img = port.random_image_u8(7000 + w, w, h)
            kps = np.array([[46.0, 46.0, 0.0, 0.0], [w - 47.0, h - 47.0, 2.5, 0.0], [46.0, h - 47.0, -1.0, 0.0],
                            [w - 47.0, 46.0, 0.7, 0.0], [45.999, 46.0, 0.0, 0.0], [w / 2, h / 2, 3.1, 0.0]])
            kept_idx, want = port.describe_all(img.astype(np.float64), kps)
            assert 4 <= len(kept_idx) <= 5 and 4 not in kept_idx        # (45.999, 46) violates the margin
            assert np.array_equal(lk.describe(img, kps)[1], want), (w, h, "host u8")
            assert np.array_equal(lk.describe(img.astype(np.float64), kps)[1], want), (w, h, "host f64")
            xycs, kept = eng.prepare_keypoints(kps, w, h)
            d_img = torch.from_numpy(img).cuda()                    # pitch == width: unaligned rows
            got = eng.extract_device(d_img, torch.from_numpy(xycs).cuda())
            torch.cuda.synchronize()
            assert np.array_equal(got.cpu().numpy(), want), (w, h, "device tensor")
            d_odd = torch.from_numpy(np.pad(img, ((0, 0), (3, 0))))[:, 3:].cuda()   # contiguous copy, odd base offset
            got = eng.extract_device(d_odd.contiguous(), torch.from_numpy(xycs).cuda())
            torch.cuda.synchronize()
            assert np.array_equal(got.cpu().numpy(), want), (w, h, "device tensor 2")
    finally:
        eng.set_option("extract_variant", 5)


def _near_tie_images(w, h):
    """u8 images built to put d1 - d2 at or next to zero: the inputs on which an fp32 estimate
    of the SSD pair must NOT be trusted (exact ties, rounding-level differences, tiny sums)."""
    rng = np.random.default_rng(1609)
    yy, xx = np.mgrid[0:h, 0:w]
    out = {
        "flat": np.full((h, w), 200, np.uint8),
        "black": np.zeros((h, w), np.uint8),
        "white": np.full((h, w), 255, np.uint8),
        "lsb_noise": (128 + rng.integers(0, 2, (h, w))).astype(np.uint8),
        "pm1_noise": (17 + rng.integers(-1, 2, (h, w))).astype(np.uint8),
        "ramp_x": (xx % 256).astype(np.uint8),
        "ramp_diag": ((xx + 2 * yy) // 3 % 256).astype(np.uint8),
        "checker8": (((xx // 8 + yy // 8) % 2) * 255).astype(np.uint8),
        "stripes4": (((xx // 4) % 2) * 90 + 40).astype(np.uint8),
        "half_flat": np.where(xx < w // 2, 255, rng.integers(0, 256, (h, w))).astype(np.uint8),
        "blocks": (rng.integers(0, 4, (h // 16 + 1, w // 16 + 1)) * 85).astype(np.uint8)
                  .repeat(16, 0).repeat(16, 1)[:h, :w],
        "sparse_dots": np.where(rng.random((h, w)) < 0.01, 255, 0).astype(np.uint8),
    }
    return out


@pytest.mark.parametrize("variant", [2, 3, 4, 5, 6])
def test_filtered_kernel_on_near_ties(lk, port, variant):
    """The filtered and pipelined kernels decide a bit from fp32 sums only when a rigorous error bound
    separates them; everything else is recomputed in exact fp64. Flat regions, periodic
    patterns and one-grey-level noise make ties and rounding-level differences the common case:
    descriptors must still be the oracle's, for axis-aligned and arbitrary angles."""
    eng = lk.get_engine()
    eng.set_option("extract_variant", variant)
    w, h = 320, 240
    kps = port.random_keypoints(77, w, h, 150)
    kps[::3, 2] = 0.0                            # upright windows: samples land on pixel centres +- 0.5
    kps[1::7, 2] = np.pi / 2
    kps[::5, :2] = np.floor(kps[::5, :2]) + 0.5  # half-integer centres: samples exactly on pixels
    for name, img in _near_tie_images(w, h).items():
        want = port.describe_all(img.astype(np.float64), kps)[1]
        got = lk.describe(img, kps)[1]
        assert np.array_equal(got, want), name
        assert np.array_equal(lk.describe(img.astype(np.float64), kps)[1], want), (name, "f64")
    eng.set_option("extract_variant", 5)


@pytest.mark.parametrize("variant", [2, 3, 4, 5, 6])
def test_filtered_kernel_exact_pass_rate(lk, port, variant):
    """Diagnostics counters: on noise the exact pass is rare (that is where the speed comes
    from), on a flat image every triplet takes it (that is where the exactness comes from)."""
    eng = lk.get_engine()
    eng.set_option("extract_variant", variant)
    w, h, n = 640, 480, 2000
    kps = port.random_keypoints(1610, w, h, n)
    try:
        eng.set_option("extract_stats", 1)
        noise = port.random_image_u8(1609, w, h)
        m = len(lk.describe(noise, kps)[1])
        exact, _ = eng.extract_stats()
        assert exact < (3e-3 if variant >= 5 else 1e-3) * m * 512, exact   # 16-bit planes: a looser bound, ~6e-4
        eng.set_option("extract_stats", 1)       # re-arm: zeroes the counters
        lk.describe(np.full((h, w), 31, np.uint8), kps)
        exact, passes = eng.extract_stats()      # passes: warps (variant 2) / windows re-resampled (3)
        assert exact == m * 512 and passes > 0
    finally:
        eng.set_option("extract_stats", 0)
        eng.set_option("extract_variant", 5)


def test_sparse_undecided_bits_are_parked_and_recomputed_exactly(lk, port):
    """Default kernel: a quad with only a few undecided triplets parks them and the whole CTA recomputes
    each one exactly after its pipeline has drained (no window-wide pass, no stall). Images where that is
    the common case — noise with a few saturated blobs, isolated flat patches — must give the oracle's
    descriptors, the counters must show parked bits, and scattered output rows (banded float64 upload)
    must be patched in the right place."""
    eng = lk.get_engine()
    w, h, n = 1024, 768, 6000
    rng = np.random.default_rng(20261017)
    yy, xx = np.mgrid[0:h, 0:w]
    noise = port.random_image_u8(4242, w, h)
    blobs = noise.copy()
    for _ in range(160):                                   # small saturated discs: ties inside, texture around
        cy, cx, r = rng.integers(0, h), rng.integers(0, w), rng.integers(5, 12)
        blobs[(yy - cy) ** 2 + (xx - cx) ** 2 <= r * r] = 255
    kps = port.random_keypoints(4243, w, h, n)
    try:
        for name, img in (("noise", noise), ("blobs", blobs)):
            want = port.describe_all(img.astype(np.float64), kps)[1]
            eng.set_option("extract_stats", 1)
            got = lk.describe(img, kps)[1]
            exact, window_passes = eng.extract_stats()
            assert np.array_equal(got, want), name
            assert exact > 0, (name, "no undecided bit at all: the test image is too tame")
            if name == "noise":
                assert window_passes == 0, (name, exact, window_passes)   # every undecided bit was parked
            eng.set_option("extract_stats", 0)
            f64 = np.ascontiguousarray(img, dtype=np.float64)           # banded upload: out_index rows
            eng.set_option("host_promote", 2)                           # (the doubles go up, the device classifies)
            for bands in (1, 3):
                eng.set_option("upload_bands", bands)
                assert np.array_equal(lk.describe(f64, kps)[1], want), (name, bands)
    finally:
        eng.set_option("extract_stats", 0)
        eng.set_option("upload_bands", 0)
        eng.set_option("host_promote", 0)


def test_estimate_planes_stay_within_the_error_budget(lk, port):
    """The default kernel decides a bit from 16-bit samples that its fp32 / fixed-point resampler produces, and its error
    bound (csrc/clatch_extract.cu) rests on one measurable claim: every stored sample A is within 0.66 units of 256 x
    the reference's window value (rounding 0.5 + resampling 0.16). clatch_estimate_planes_u8_dev returns those samples
    from the production resampler; here every sample of every window — noise, hard edges, ramps, saturated blocks,
    upright / half-integer / arbitrary keypoints — is held against the oracle's extract_window."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_pattern(None)                  # (the entry point only needs some pattern to be installed)
    w, h, n = 640, 480, 220
    rng = np.random.default_rng(66)
    yy, xx = np.mgrid[0:h, 0:w]
    images = {
        "noise": port.random_image_u8(660, w, h),
        "checker3": (((xx // 3 + yy // 3) % 2) * 255).astype(np.uint8),            # the steepest slopes there are
        "ramp": ((xx * 3 + yy) % 256).astype(np.uint8),
        "blocks": (rng.integers(0, 2, (h // 16 + 1, w // 16 + 1)) * 255).astype(np.uint8).repeat(16, 0).repeat(16, 1)[:h, :w],
        "structured": port.structured_image(661, w, h).astype(np.uint8),
    }
    kps = port.random_keypoints(662, w, h, n)
    kps[::4, 2] = 0.0
    kps[1::8, 2] = np.pi / 2
    kps[::5, :2] = np.floor(kps[::5, :2]) + 0.5
    kps[3::7, :2] = np.floor(kps[3::7, :2])
    xycs, kept = eng.prepare_keypoints(kps, w, h)
    d_x = torch.from_numpy(xycs).cuda()
    worst = 0.0
    for name, img in images.items():
        planes = eng.estimate_planes_device(torch.from_numpy(img).cuda(), d_x)
        torch.cuda.synchronize()
        got = planes.cpu().numpy().view(np.uint16).astype(np.float64)
        f64 = img.astype(np.float64)
        for j, i in enumerate(kept):
            want = 256.0 * np.asarray(port.extract_window(f64, kps[i])).reshape(64, 64)
            err = np.abs(got[j] - want).max()
            worst = max(worst, err)
            assert err <= 0.66, (name, j, err)
    assert worst > 0.4            # (rounding alone reaches 0.5: the check is not vacuous)
    print(f"largest |A - 256 v| over {len(images) * len(kept)} windows: {worst:.4f} of the 0.66 budgeted")


def test_float64_images_through_the_packed_plane_kernel(lk, port):
    """A float64 image that is not u8-valued but tame (finite, a value range between 2^-400 and 2^400, no pixel further than
    2^20 ranges from zero) takes the default kernel as well: its estimate planes come from a float texture of the image scaled to [0, 1]
    over its own range, every undecided bit is recomputed from the doubles in global memory. Anything else (flat,
    a ripple on a huge offset) stays with the all-fp64 kernel. Either way the descriptors are the oracle's — through
    describe(), a device tensor and describe_batch(), with the route switched on and off."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    w, h, n = 640, 400, 1500
    rng = np.random.default_rng(31)
    yy, xx = np.mgrid[0:h, 0:w]
    noise = rng.random((h, w))
    blocks = np.where(((xx // 24) + (yy // 24)) % 2 == 0, 0.5, 200.25)          # two levels: ties everywhere inside a block
    images = {
        "noise x 255": (noise * 255.0, True),
        "negative": (noise * 300.0 - 128.5, True),
        "ramp with repeats": ((xx * 0.37 + yy * 0.11) % 50.0, True),
        "two levels": (blocks, True),
        "two levels + speckle": (np.where(rng.random((h, w)) < 0.02, noise * 255.0, blocks), True),
        "offset 1e5": (1.0e5 + noise, True),
        "small values": (noise * 3.0e-100 + 1.0e-101, True),
        "tiny values": (noise * 3.0e-290 + 1.0e-291, False),                     # the reference's squares underflow: every bit 0
        "big values": (noise * 3.0e200, False),                                  # ... or overflow
        "offset 1e9": (1.0e9 + noise, False),                                    # further than 2^20 ranges from zero
        "flat": (np.full((h, w), 100.5), False),
        "nearly flat": (100.5 + 1.0e-12 * noise, False),
    }
    kps = port.random_keypoints(32, w, h, n)
    kps[::4, 2] = 0.0
    kps[::9, :2] = np.floor(kps[::9, :2]) + 0.5
    try:
        for name, (img, routed) in images.items():
            want = port.describe_all(img, kps)[1]
            eng.set_option("extract_stats", 1)
            got = lk.describe(img, kps)[1]
            exact, _ = eng.extract_stats()
            eng.set_option("extract_stats", 0)
            assert np.array_equal(got, want), name
            if name.startswith("two levels"):
                assert exact > 0, name                 # the estimate-based kernel ran (the all-fp64 kernel counts nothing)
            if not routed:
                assert exact == 0, name
            xycs, _ = eng.prepare_keypoints(kps, w, h)
            dev = eng.extract_device(torch.from_numpy(img).cuda(), torch.from_numpy(xycs).cuda())
            torch.cuda.synchronize()
            assert np.array_equal(dev.cpu().numpy(), want), (name, "device tensor")
            eng.set_option("extract_f64_h16", 0)
            assert np.array_equal(lk.describe(img, kps)[1], want), (name, "route off")
            eng.set_option("extract_f64_h16", 1)
        # a frame big enough (>= 4 MB) for the host paths that only big frames take: the probe that sends a visibly
        # non-u8 frame up in one piece, and the chunked page-locked staging of frames in ordinary numpy memory
        big = rng.random((800, 1100)) * 200.0 + 3.5
        big_kps = port.random_keypoints(33, 1100, 800, 5000)
        want_big = port.describe_all(big, big_kps)[1]
        assert np.array_equal(lk.describe(big, big_kps)[1], want_big), "big pageable frame"
        pin = torch.empty(big.shape, dtype=torch.float64, pin_memory=True)
        pin.numpy()[...] = big
        assert np.array_equal(lk.describe(pin.numpy(), big_kps)[1], want_big), "big page-locked frame"
        big_int = np.floor(big)                                                   # u8-valued: the banded upload, u8 kernels
        assert np.array_equal(lk.describe(big_int, big_kps)[1], port.describe_all(big_int, big_kps)[1]), "big u8-valued frame"
        names = ["noise x 255", "two levels", "flat", "negative"]
        res = lk.describe_batch([images[k][0] for k in names], [kps] * len(names))
        for k, (_, desc) in zip(names, res):
            assert np.array_equal(desc, port.describe_all(images[k][0], kps)[1]), (k, "batch")
    finally:
        eng.set_option("extract_stats", 0)
        eng.set_option("extract_f64_h16", 1)


@pytest.mark.parametrize("promote", [1, 2, 0])
def test_float64_promotion_edges(lk, port, promote):
    """A float64 image goes to the u8 kernels only if EVERY pixel is an integer in [0, 255] (host
    workers or device classifier, same rule). One odd pixel anywhere — vector body, scalar tail,
    first or last row — must send the whole image down the float64 route, and either way the
    descriptors are the oracle's. host_promote 1 = host workers always, 2 = device classifier always,
    0 = host workers for ordinary numpy memory (what this test passes)."""
    eng = lk.get_engine()
    eng.set_option("host_promote", promote)
    try:
        w, h = 331, 207                                   # width % 8 != 0: exercises the scalar tail
        base = port.random_image_u8(321, w, h).astype(np.float64)
        kps = port.random_keypoints(322, w, h, 300)
        want = port.describe_all(base, kps)[1]
        assert np.array_equal(lk.describe(base, kps)[1], want)
        neg_zero = base.copy()
        neg_zero[base == 0] = -0.0                        # still u8-valued
        assert np.array_equal(lk.describe(neg_zero, kps)[1], want)
        for (y, x), v in {(0, 0): 100.5, (h - 1, w - 1): 256.0, (100, 328): -1.0, (57, 160): 1e300,
                          (101, 7): 254.99999999999997, (h // 2, 3): 2.0 ** -40}.items():
            img = base.copy()
            img[y, x] = v
            assert np.array_equal(lk.describe(img, kps)[1], port.describe_all(img, kps)[1]), (y, x, v)
    finally:
        eng.set_option("host_promote", 0)


@pytest.mark.parametrize("bands", [1, 2, 3, 6])
def test_banded_float64_upload(lk, port, bands):
    """A big float64 frame goes up in row bands and each band's keypoints are extracted while the
    next band is in flight; descriptors come back in input order. u8-valued frames take the u8
    kernel band by band, a frame that stops being u8-valued in a later band switches to the
    float64 kernel from that band on, and a non-integer frame uses it throughout — always the
    oracle's bytes, including margin violators and keypoints on band boundaries."""
    eng = lk.get_engine()
    eng.set_option("upload_bands", bands)
    eng.set_option("host_promote", 2)            # numpy memory would otherwise be promoted on the host, not banded
    try:
        w, h, n = 1024, 768, 6000
        base = port.random_image_u8(8100, w, h).astype(np.float64)
        kps = port.random_keypoints(8101, w, h, n)
        kps[::97, 0] = 3.0                                             # margin violators are dropped silently
        edge_rows = [h // bands * b for b in range(1, bands)] or [h // 2]
        for i, r in enumerate(edge_rows):                              # footprints ending exactly at band edges
            kps[10 + i, 1] = r - 46.0
            kps[40 + i, 1] = r - 47.0 + 0.999
            kps[70 + i, 1] = r - 45.5
        late = base.copy()
        late[h - 5, w // 2] = 17.25                                    # not u8-valued, but only in the last rows
        frac = base + np.random.default_rng(3).random(base.shape) * 0.5
        for name, img in (("u8-valued", base), ("late non-integer pixel", late), ("non-integer", frac)):
            kept_idx, want = port.describe_all(img, kps)
            kept, desc = lk.describe(img, kps)
            assert np.array_equal(kept, kps[kept_idx]), name
            assert np.array_equal(desc, want), name
    finally:
        eng.set_option("upload_bands", 0)
        eng.set_option("host_promote", 0)


# ------------------------------------------------------ resident sets, batched pairs ----

@pytest.mark.parametrize("filter_on_device,cta_pairs", [(1, 1), (0, 1), (1, 0)])
def test_resident_sets_and_batched_pairs(lk, port, filter_on_device, cta_pairs):
    """cfg5 shape: every image against every other image through resident descriptor sets.
    Each pair must equal the reference's match_brute_force with the same filters, whether the
    filter pass (ratio in double, inclusive max distance, cross-check) runs on the device or the host."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_option("pairs_filter_on_device", filter_on_device)
    eng.set_option("match_pairs", cta_pairs)      # item tables in CTA-pair form (fillers for odd tile counts) or plain
    sizes = [300, 1, 257, 128, 1000]
    raw = [port.random_descriptors(900 + i, n, 64) for i, n in enumerate(sizes)]
    raw[2][5] = raw[0][7]                 # cross-image duplicates -> zero distances and ties
    raw[4][11] = raw[0][7]
    raw[4][12] = raw[4][11]
    sets = [eng.create_set(raw[0]), eng.create_set(torch.from_numpy(raw[1]).cuda()), eng.create_set(raw[2]),
            eng.create_set(torch.from_numpy(raw[3]).cuda()), eng.create_set(raw[4])]
    assert [len(s) for s in sets] == sizes
    pairs = [(i, j) for i in range(5) for j in range(5) if i != j]
    for kw in ({}, {"ratio": 0.9}, {"cross_check": True}, {"ratio": 0.85, "cross_check": True, "max_distance": 240},
               {"ratio": 1.0, "max_distance": 0}, {"ratio": float("inf")}, {"ratio": float("nan")}, {"max_distance": -1}):
        got = eng.match_set_pairs(sets, pairs, **kw)
        for (i, j), g in zip(pairs, got):
            assert np.array_equal(g, port.match(raw[i], raw[j], **kw)), (i, j, kw)
    one = eng.match_sets(sets[0], sets[4], ratio=0.9, cross_check=True)
    assert np.array_equal(one, port.match(raw[0], raw[4], ratio=0.9, cross_check=True))
    assert eng.match_set_pairs(sets, []) == []
    empty = eng.create_set(np.zeros((0, 64), np.uint8))
    assert len(eng.match_sets(empty, sets[0])) == 0            # empty probes -> no rows
    with pytest.raises(RuntimeError):
        eng.match_sets(sets[0], empty)                          # empty gallery -> EmptyGallery
    for s in sets:
        s.close()
    # the sharded driver's single-process form
    from paper_1609_03986_b200 import sharded
    res = sharded.match_all_pairs_resident(raw, ratio=0.9, cross_check=True)
    assert sorted(res) == sharded.pairs_for_rank(5, 0, 1)
    for (i, j), m in res.items():
        assert np.array_equal(m, port.match(raw[i], raw[j], ratio=0.9, cross_check=True))
    eng.set_option("pairs_filter_on_device", 1)
    eng.set_option("match_pairs", 1)


def test_result_arrays_are_never_recycled_while_alive(lk, port):
    """describe() hands back page-locked arrays from a recycling pool: a block may be reused only
    after the last view of it is gone. Results that are kept must keep their contents."""
    import gc
    w, h = 320, 240
    imgs = [port.random_image_u8(4000 + i, w, h) for i in range(12)]
    kps = port.random_keypoints(4100, w, h, 400)
    want = [port.describe_all(im.astype(np.float64), kps)[1] for im in imgs]
    kept = []
    for i, im in enumerate(imgs):                  # keep every other result (through a slice view), drop the rest
        d = lk.describe(im, kps)[1]
        assert np.array_equal(d, want[i])
        if i % 2 == 0:
            kept.append((i, d[3:]))
        del d
        gc.collect()
    for i, view in kept:
        assert np.array_equal(view, want[i][3:]), i
    batch = lk.describe_batch(imgs[:5], [kps] * 5)
    for i, view in kept:
        assert np.array_equal(view, want[i][3:]), i
    for i, (_, d) in enumerate(batch):
        assert np.array_equal(d, want[i])


def test_describe_batch_matches_per_image_calls(lk, port):
    """cfg3 shape: several images per GPU through the pipelined batch call."""
    imgs, kps = [], []
    for i, (w, h, n) in enumerate([(320, 240, 500), (200, 150, 1), (640, 480, 2000), (333, 201, 0), (256, 256, 77)]):
        imgs.append(port.structured_image(600 + i, w, h) if i % 2 else port.random_image(600 + i, w, h))
        k = port.random_keypoints(700 + i, w, h, n)
        if n > 10:
            k[::9, 0] = 5.0                       # margin violators
        kps.append(k)
    want = [port.describe_all(im, k) for im, k in zip(imgs, kps)]
    for cast in (np.uint8, np.float64):
        got = lk.describe_batch([im.astype(cast) for im in imgs], kps)
        assert len(got) == len(imgs)
        for (gk, gd), (wk, wd), k in zip(got, want, kps):
            assert np.array_equal(gk, k[wk]) and np.array_equal(gd, wd)
    # non-integer images cannot be promoted to u8: the f64 sampling path inside the pipeline
    rng = np.random.default_rng(5)
    fimgs = [rng.random((150, 170)) * 255.0 for _ in range(3)]
    fk = [port.random_keypoints(800 + i, 170, 150, 90) for i in range(3)]
    for (gk, gd), im, k in zip(lk.describe_batch(fimgs, fk), fimgs, fk):
        assert np.array_equal(gd, port.describe_all(im, k)[1])
    assert lk.describe_batch([], []) == []


# ------------------------------------------------------------------- detection ----

def test_detect_golden_keypoints(lk, golden_image_u8):
    # acceptance.cpp:120-123: detect_and_orient(golden, 20, nms) is pinned by golden_keypoints.tsv
    want = np.load(GOLDEN / "golden_keypoints_f64.npy")
    for img in (golden_image_u8, golden_image_u8.astype(np.float64)):
        got = lk.detect(img, threshold=20.0)
        assert got.dtype == np.float64 and np.array_equal(got, want)


def test_detect_reference_vectors(lk, port, vectors):
    for tag, maker, args, thr, nms, ori in [("struct", "structured_image", (1, 160, 120), 20.0, True, True),
                                            ("noise", "random_image", (2, 96, 80), 30.5, True, True),
                                            ("nonms", "random_image", (3, 64, 48), 12.25, False, False)]:
        img = getattr(port, maker)(*args)
        for im in (img, img.astype(np.uint8)):
            assert np.array_equal(lk.detect(im, thr, nms, ori), vectors[f"det_{tag}_out"]), tag
    assert np.array_equal(lk.detect(vectors["det_frac_image"], 40.0), vectors["det_frac_out"])


def test_detect_against_oracle_and_edge_cases(lk, port):
    for seed, (w, h), thr, nms, ori in [(5, (640, 480), 20.0, True, True), (6, (333, 201), 25.5, False, True),
                                        (7, (97, 61), 20.0, True, False), (8, (1920, 1080), 20.0, True, True)]:
        img = port.structured_image(seed, w, h) if seed != 6 else port.random_image(seed, w, h)
        want = port.detect(img, thr, nms, ori)
        assert np.array_equal(lk.detect(img.astype(np.uint8), thr, nms, ori), want), (seed, "u8")
        assert np.array_equal(lk.detect(img, thr, nms, ori), want), (seed, "f64")
    # test_detect.cpp:34-41: uniform image -> nothing; too small -> ImageTooSmall
    assert lk.detect(np.full((32, 32), 77.0)).shape == (0, 4)
    with pytest.raises(RuntimeError):
        lk.detect(np.zeros((32, 6)))
    with pytest.raises(ValueError):
        lk.detect(np.zeros(16))
    # test_detect.cpp:43-74: bright square corners fire
    sq = np.zeros((32, 32))
    sq[12:20, 12:20] = 255.0
    got = lk.detect(sq, 20.0, nms=False, orient=False)
    assert np.array_equal(got, port.detect(sq, 20.0, False, False)) and len(got) > 0
    # detect -> describe -> match chain on the GPU (python/test_smoke.py:30-53)
    img = port.structured_image(11, 400, 300)
    kps = lk.detect(img)
    kept, desc = lk.describe(img, kps)
    assert np.array_equal(desc, port.describe_all(img, kps)[1]) and len(desc) > 0
    m = lk.match(desc, desc)
    assert np.all(m[:, 2] == 0)


# ------------------------------------------------------------ trainer scoring ----

def test_triplet_bits_scoring(lk, port, vectors):
    """select_triplets' parallel body (src/pattern.cpp:340-346,397-400) on the GPU."""
    eng = lk.get_engine()
    wins = np.stack([port.random_image(300 + i, 64, 64) for i in range(45)])
    wins[40:] = np.stack([port.structured_image(400 + i, 64, 64) for i in range(5)])
    _, _, _, seven = oracle.default_pattern()
    assert np.array_equal(eng.triplet_bits(wins, vectors["score_candidates_k8"], 8, seven), vectors["score_bits_seven"])
    assert np.array_equal(eng.triplet_bits(wins, vectors["score_candidates_k8"], 8), vectors["score_bits_ones"])
    assert np.array_equal(eng.triplet_bits(wins, vectors["score_candidates_k5"], 5, vectors["score_weights_k5"]),
                          vectors["score_bits_k5"])
    # larger, ragged sizes against the oracle (n and C not multiples of 32)
    rng = np.random.default_rng(3)
    big = np.stack([port.random_image(900 + i, 64, 64) for i in range(77)])
    cand = rng.integers(0, 57, size=(1001, 6)).astype(np.int16)
    assert np.array_equal(eng.triplet_bits(big, cand, 8, seven), port.triplet_bits(big, cand, 8, seven))
    with pytest.raises(RuntimeError):
        eng.triplet_bits(big, np.full((1, 6), 60, np.int16), 8)      # coordinate outside [0, 64-K]
    assert eng.triplet_bits(big[:0], cand, 8).shape == (1001, 0)
    # the extraction pattern is untouched by scoring (separate constant bank)
    img = port.structured_image(5, 200, 150)
    kps = port.random_keypoints(6, 200, 150, 20)
    assert np.array_equal(lk.describe(img, kps, pattern=(GOLDEN / "pattern_t64k5w.latchpat").read_text())[1],
                          port.describe_all(img, kps, pattern=oracle.parse_pattern_text(
                              (GOLDEN / "pattern_t64k5w.latchpat").read_text()))[1])


@pytest.mark.parametrize("bands", ["1", "3"])
def test_banded_upload_large_images(lk, port, bands, monkeypatch):
    """CLATCH_UPLOAD_BANDS: the image can go up in row bands with extraction queued per band;
    keypoints are bucketed by band and un-permuted on the way out. Results and order must not
    change."""
    monkeypatch.setenv("CLATCH_UPLOAD_BANDS", bands)
    eng = lk.get_engine()
    eng.set_option("host_promote", 2)                         # keep pageable float64 frames on the banded route
    w, h = 1920, 1080
    img = port.structured_image(77, w, h)                     # float64, 16.6 MB
    kps = port.random_keypoints(78, w, h, 2500)
    kps[::50, 1] = 30.0                                       # margin violators stay dropped, order kept
    kps[5] = [100.0, 46.0, 0.3, 1.0]                          # footprint ends in the first band
    kps[6] = [100.0, h - 47.0, -0.3, 2.0]                     # ... and in the last one
    want_kept, want = port.describe_all(img, kps)
    kept, desc = lk.describe(img, kps)
    assert np.array_equal(kept, kps[want_kept]) and np.array_equal(desc, want)
    frac = img + 0.25                                         # non-integer: f64 sampling kernel per band
    assert np.array_equal(lk.describe(frac, kps)[1], port.describe_all(frac, kps)[1])
    frac2 = img.copy()
    frac2[h - 3, w - 3] = 0.5                                 # only the LAST band is non-integer
    assert np.array_equal(lk.describe(frac2, kps)[1], port.describe_all(frac2, kps)[1])
    big = port.random_image_u8(79, 3840, 2160)                # uint8, 8.3 MB
    k2 = port.random_keypoints(80, 3840, 2160, 2100)
    assert np.array_equal(lk.describe(big, k2)[1], port.describe_all(big.astype(np.float64), k2)[1])
    eng.set_option("host_promote", 0)


# ------------------------------------------- round-2 additions: semantics at the edges ----

def _nonfinite_cases(base, kps):
    """Images with NaN / Inf / overflowing pixels placed under LIVE patch pixels and under the mask's
    zero-weight row 7 / column 7 of some triplet's patches (src/descriptor.cpp:66-71: w*e*e with w = 0
    and e = NaN still poisons the sum, so the bit must come out 0 exactly as the reference computes it)."""
    h, w = base.shape
    x, y = int(kps[0, 0]), int(kps[0, 1])
    cases = {}
    for name, v in (("nan", np.nan), ("inf", np.inf), ("-inf", -np.inf)):
        for where, (dy, dx) in (("centre", (0, 0)), ("edge", (-31, 24)), ("far", (20, -30))):
            img = base.copy()
            img[y + dy, x + dx] = v
            cases[f"{name}@{where}"] = img
    img = base.copy()
    img[y, x], img[y + 1, x] = 1.5e308, -1.5e308            # finite pixels whose difference overflows
    cases["overflowing difference"] = img
    img = base.copy()
    img[::37, ::41] = np.nan                                 # scattered: most windows hold a NaN somewhere
    cases["scattered nan"] = img
    img = base.copy()
    img[y - 3:y + 3, x - 3:x + 3] = 2.0 ** 1001              # huge but finite
    cases["huge block"] = img
    return cases


def test_nonfinite_pixels_follow_the_reference(lk, port):
    w, h = 400, 300
    base = port.structured_image(66, w, h)
    kps = port.random_keypoints(67, w, h, 500)
    kps[0] = [200.0, 150.0, 0.0, 0.0]                        # upright, integer centre: samples ARE pixels
    kps[1] = [200.5, 150.5, 0.7, 0.0]
    ref = oracle.ref()
    with np.errstate(all="ignore"):
        for name, img in _nonfinite_cases(base, kps).items():
            want = port.describe_all(img, kps)[1]
            if ref is not None:
                assert np.array_equal(ref.describe_all(img, kps, workers=0)[1], want), name
            assert np.array_equal(lk.describe(img, kps)[1], want), name
            assert not np.array_equal(want, port.describe_all(base, kps)[1])
            got_b = lk.describe_batch([img, base], [kps, kps])
            assert np.array_equal(got_b[0][1], want) and np.array_equal(got_b[1][1], port.describe_all(base, kps)[1])


def test_nonfinite_pixels_banded_and_device(lk, port):
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    w, h, n = 1024, 768, 5000
    base = port.random_image_u8(8100, w, h).astype(np.float64)
    kps = port.random_keypoints(8101, w, h, n)
    img = base.copy()
    img[h - 60, w // 2] = np.nan                             # only the LAST band sees it
    img[100, 100] = np.inf
    want = port.describe_all(img, kps)[1]
    with np.errstate(all="ignore"):
        for promote in (2, 0):                               # banded device route, host-promote attempt then device
            eng.set_option("host_promote", promote)
            try:
                assert np.array_equal(lk.describe(img, kps)[1], want)
            finally:
                eng.set_option("host_promote", 0)
    xycs, kept = eng.prepare_keypoints(kps, w, h)
    out = eng.extract_device(torch.from_numpy(img).cuda(), torch.from_numpy(xycs).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)


def test_negative_and_odd_strides(lk, port):
    """Views the reference accepts through its c_style | forcecast conversion (bindings/module.cpp:30):
    flipped, transposed, broadcast and row-skipping arrays, uint8 and float64."""
    img8 = port.random_image_u8(91, 300, 200)
    for base in (img8, img8.astype(np.float64)):
        views = (base[::-1], base[:, ::-1], base.T[:, :200], np.broadcast_to(base[50], (200, 300)), base[::2, 1:],
                 base[::-1, ::-1][3:])
        for v in views:
            flat = np.ascontiguousarray(v)
            hh, ww = flat.shape
            k = port.random_keypoints(93, ww, hh, 60)
            assert np.array_equal(lk.describe(v, k)[1], port.describe_all(flat.astype(np.float64), k)[1]), v.strides
    assert np.array_equal(lk.detect(img8[::-1]), lk.detect(np.ascontiguousarray(img8[::-1])))


def test_concurrent_callers_with_different_patterns(lk, port):
    """describe() is a pure function in the reference; here the pattern is context state, so it is
    installed under the same lock as the launch. Threads with different patterns never see each other's."""
    import threading
    img = port.structured_image(97, 140, 140)
    kps = port.random_keypoints(98, 140, 140, 64)
    texts = [None, (GOLDEN / "pattern_t8k8.latchpat").read_text(), (GOLDEN / "pattern_t64k5w.latchpat").read_text()]
    want = [lk.describe(img, kps, pattern=t)[1] for t in texts]
    assert len({w.shape[1] for w in want}) == 3
    errors = []

    def worker(i):
        try:
            for _ in range(40):
                got = lk.describe(img, kps, pattern=texts[i])[1]
                if not np.array_equal(got, want[i]):
                    errors.append(f"thread {i}: wrong pattern's descriptors ({got.shape})")
                    return
        except Exception as exc:                              # noqa: BLE001
            errors.append(f"thread {i}: {type(exc).__name__}: {exc}")
    threads = [threading.Thread(target=worker, args=(i,)) for i in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_device_calls_on_different_streams_share_scratch_safely(lk, port):
    """clatch_match_top2_dev / clatch_extract_f64_dev queue on the caller's stream but use the context's
    expanded-operand and partial buffers: calls on different streams must be ordered by the library."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_pattern(None)                                # extract_device uses the context's installed pattern
    sets = [torch.from_numpy(port.random_descriptors(200 + i, 6000 + 500 * i, 64)).cuda() for i in range(4)]
    want = [port.knn2_all(s.cpu().numpy()[:3000], s.cpu().numpy()).T for s in sets]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(6):
        outs = []
        for i, s in enumerate(sets):
            st = streams[i & 1]
            with torch.cuda.stream(st):
                outs.append(eng.match_top2_device(s[:3000], s, stream=st))
        bi, bd, sd = eng.match_top2(sets[0].cpu().numpy()[:100], sets[1].cpu().numpy())     # host form in between
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert np.array_equal(o.cpu().numpy(), w), rep
    w, h = 640, 480
    imgs = [port.random_image_u8(300 + i, w, h).astype(np.float64) for i in range(2)]
    imgs[1] += 0.25                                          # one u8-valued, one not: different flag values
    kps = port.random_keypoints(310, w, h, 800)
    xycs, _ = eng.prepare_keypoints(kps, w, h)
    d_x = torch.from_numpy(xycs).cuda()
    d_imgs = [torch.from_numpy(a).cuda() for a in imgs]
    wants = [port.describe_all(a, kps)[1] for a in imgs]
    torch.cuda.synchronize()
    for rep in range(4):
        outs = []
        for i in (0, 1, 0, 1):
            with torch.cuda.stream(streams[i]):
                outs.append((i, eng.extract_device(d_imgs[i], d_x, stream=streams[i])))
        torch.cuda.synchronize()
        for i, o in outs:
            assert np.array_equal(o.cpu().numpy(), wants[i]), (rep, i)


def test_pageable_float64_batch_is_promoted_on_the_host(lk, port):
    """describe_batch on ordinary numpy float64 frames: u8-valued frames are converted by the host workers
    into page-locked staging and go up as bytes; a frame with one odd pixel takes the float64 route."""
    imgs = [port.random_image_u8(400 + i, 800, 600).astype(np.float64) for i in range(4)]
    imgs[2][599, 799] = 0.5
    imgs[3][0, 0] = np.nan
    kps = [port.random_keypoints(410 + i, 800, 600, 700) for i in range(4)]
    with np.errstate(all="ignore"):
        want = [port.describe_all(a, k)[1] for a, k in zip(imgs, kps)]
        for promote in (0, 1, 2):
            lk.get_engine().set_option("host_promote", promote)
            try:
                got = lk.describe_batch(imgs, kps)
            finally:
                lk.get_engine().set_option("host_promote", 0)
            for g, wnt in zip(got, want):
                assert np.array_equal(g[1], wnt), promote


def test_tensor_matcher_extreme_distances(lk, port):
    """The tensor-core matcher over the whole distance range: identical rows (D = +512), complements
    (D = -512), all-zero / all-one descriptors, ties on tile boundaries, graded small distances."""
    eng = lk.get_engine()
    rng = np.random.default_rng(16)
    train = port.random_descriptors(77, 3000)
    train[0] = 0
    train[1] = 255
    train[2] = ~train[5]
    train[2999] = train[5]
    query = port.random_descriptors(78, 700)
    query[0] = 0
    query[1] = 255
    query[2] = train[5]                                  # exact copy, twice in train (5 and 2999)
    query[3] = ~train[7]                                 # complement: distance 512 to row 7
    for k in range(4, 40):                               # graded distances 0..35 from train[100 + k]
        query[k] = train[100 + k]
        for b in rng.choice(512, k - 4, replace=False):
            query[k, b >> 3] ^= np.uint8(1 << (b & 7))
    only = np.stack([train[7], train[7]])                # every distance 512 for query 3
    got = np.stack(eng.match_top2(query, train), 1)
    assert np.array_equal(got, port.knn2_all(query, train))
    assert got[2].tolist() == [5, 0, 0] and got[0].tolist()[:2] == [0, 0] and got[1].tolist()[:2] == [1, 0]
    far = np.stack(eng.match_top2(query[3:4], only), 1)
    assert far.tolist() == [[0, 512, 512]]
    sets = [eng.create_set(query), eng.create_set(train)]
    rows = eng.match_sets(sets[0], sets[1], ratio=0.9, cross_check=True)
    assert np.array_equal(rows, port.match(query, train, ratio=0.9, cross_check=True))
    rows = eng.match_sets(sets[0], sets[1], max_distance=40)
    assert np.array_equal(rows, port.match(query, train, max_distance=40))


@pytest.mark.parametrize("q,n", [(5000, 6000), (5000, 300), (4096, 40000), (1500, 1200)])
def test_single_pair_match_filters_on_the_device(lk, port, q, n):
    """match() between two sets big enough for the device-side filter pass: cross-check between sets of
    similar size runs both passes as one launch over temporary resident sets, anything else keeps the two
    launches and filters the result block on the device. Rows must be the reference's in every combination,
    including planted duplicates (ties on both passes) and with the host filter."""
    d = port.random_descriptors(4200 + q, q + n, 64)
    probes, gallery = d[:q].copy(), d[q:].copy()
    rng = np.random.default_rng(q + n)
    rows = rng.choice(q, min(q, n) // 4, replace=False)
    gallery[rng.choice(n, len(rows), replace=False)] = probes[rows]       # true matches ...
    for r in rows[:len(rows) // 2]:                                        # ... half of them a few bits off
        for b in rng.integers(0, 512, 5):
            probes[r, b >> 3] ^= np.uint8(1 << (b & 7))
    gallery[n - 1] = gallery[0]
    probes[q - 1] = probes[1]
    eng = lk.get_engine()
    combos = ({"ratio": 0.8}, {"cross_check": True}, {"max_distance": 200}, {"ratio": 0.8, "cross_check": True},
              {"ratio": 0.9, "cross_check": True, "max_distance": 240})
    want = [port.match(probes, gallery, **kw) for kw in combos]
    assert all(len(w) > 0 for w in want)
    try:
        for on_device in (1, 0):
            eng.set_option("pairs_filter_on_device", on_device)
            for kw, w in zip(combos, want):
                assert np.array_equal(lk.match(probes, gallery, **kw), w), (on_device, kw)
    finally:
        eng.set_option("pairs_filter_on_device", 1)
    assert np.array_equal(lk.match(probes, probes, cross_check=True), port.match(probes, probes, cross_check=True))


def test_degenerate_streams_are_routed_to_the_quad_kernel_and_stay_exact(lk, port):
    """A context whose last launch needed the exact pass for more than a quarter of its windows (flat or saturated
    images) runs its next launches on the all-fp64 quad kernel and probes the default kernel again after 16 launches
    (then 32, 64, 128 while the probes agree). Whatever the router decides, and however flat and textured images alternate, the descriptors are
    the oracle's."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_pattern(None)
    w, h = 640, 480
    kps = port.random_keypoints(5151, w, h, 900)
    noise = port.random_image_u8(5150, w, h)
    flat = np.full((h, w), 77, np.uint8)
    half = noise.copy()
    half[:, : w // 2] = 255
    want = {name: port.describe_all(im.astype(np.float64), kps)[1] for name, im in (("noise", noise), ("flat", flat), ("half", half))}
    imgs = {"noise": noise, "flat": flat, "half": half}
    xycs, _ = eng.prepare_keypoints(kps, w, h)
    d_x = torch.from_numpy(xycs).cuda()
    d_imgs = {k: torch.from_numpy(v).cuda() for k, v in imgs.items()}
    order = ["flat"] * 20 + ["noise"] * 20 + ["flat", "noise", "half"] * 8
    try:
        for route in (1, 0):
            eng.set_option("extract_route", route)
            for i, name in enumerate(order):
                if i % 3 == 0:
                    got = lk.describe(imgs[name], kps)[1]
                else:
                    got = eng.extract_device(d_imgs[name], d_x)
                    torch.cuda.synchronize()
                    got = got.cpu().numpy()
                assert np.array_equal(got, want[name]), (route, i, name)
    finally:
        eng.set_option("extract_route", 1)


def test_dynamically_scheduled_quads_cover_every_keypoint_once(lk, port):
    """The default kernel hands its quads (four keypoints) out through a device counter that the last CTA to draw
    rewinds for the next launch: back-to-back launches of very different sizes — fewer quads than CTAs, exactly the
    statically assigned first three rounds, one more, many more, ragged last quads — on a clean and on a partly
    saturated image (where the window-wide pass makes the CTAs' speeds differ) must all give the oracle's bits,
    with no launch inheriting a counter that was not rewound."""
    torch = pytest.importorskip("torch")
    eng = lk.get_engine()
    eng.set_pattern(None)
    w, h = 800, 600
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    noise = port.random_image_u8(6060, w, h)
    part = noise.copy()
    part[:, : w // 6] = 255
    part[h // 2 :, w // 2 :] = 0
    sizes = [1, 3, 4, 5, 4 * sms - 1, 4 * sms, 4 * sms + 1, 12 * sms - 2, 12 * sms, 12 * sms + 1, 16 * sms + 3, 5000, 7, 4 * sms + 2, 9001]
    kps = port.random_keypoints(6061, w, h, 12000)
    xycs, _ = eng.prepare_keypoints(kps, w, h)
    assert len(xycs) >= max(sizes)
    want = {name: port.describe_all(im.astype(np.float64), kps)[1] for name, im in (("noise", noise), ("part", part))}
    d_imgs = {"noise": torch.from_numpy(noise).cuda(), "part": torch.from_numpy(part).cuda()}
    d_x = torch.from_numpy(xycs).cuda()
    try:
        eng.set_option("extract_route", 0)          # keep the default kernel on the partly saturated image too
        outs = []
        for rep in range(3):
            for i, m in enumerate(sizes):
                name = "part" if (i + rep) % 2 else "noise"
                outs.append((name, m, eng.extract_device(d_imgs[name], d_x[:m].contiguous())))   # no sync in between
        torch.cuda.synchronize()
        for name, m, got in outs:
            assert np.array_equal(got.cpu().numpy(), want[name][:m]), (name, m)
    finally:
        eng.set_option("extract_route", 1)
