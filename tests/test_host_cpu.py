"""CPU-only checks of the host side: the C-ABI library loads and exports every symbol
include/clatch.h declares, the host-only entry points (keypoint preparation, match
filter pass) agree with the oracle, the pattern reader mirrors the reference's, and
the product refuses to run without a GPU instead of falling back to anything."""
import ctypes as C
import re

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_1609_03986_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_1609_03986_b200 import _lib
    header = (ROOT / "include" / "clatch.h").read_text()
    declared = set(re.findall(r"CLATCH_API[^;(]*?\b(clatch_\w+)\s*\(", header))
    assert len(declared) >= 17
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert getattr(lib, name) is not None


def test_header_compiles_as_plain_c(tmp_path):
    import subprocess
    src = tmp_path / "t.c"
    src.write_text('#include "clatch.h"\nint main(void){return CLATCH_OK;}\n')
    subprocess.run(["/usr/bin/gcc", "-std=c99", "-pedantic", "-Werror", "-I", str(ROOT / "include"),
                    "-c", str(src), "-o", str(tmp_path / "t.o")], check=True)


def test_prepare_keypoints_matches_oracle_margin_and_libm(lib, port):
    from paper_1609_03986_b200.engine import Engine
    prep = Engine.prepare_keypoints.__get__(type("E", (), {"lib": lib})())
    w, h = 300, 200
    kps = port.random_keypoints(5, w, h, 20000)
    kps[::7, 0] -= 60.0
    kps[::11, 1] += 120.0
    kps[3] = [46.0, 46.0, 0.1, 0]
    kps[4] = [w - 47.0, h - 47.0, 0.2, 0]
    kps[5] = [w - 46.999, 60.0, 0.3, 0]
    kps[6] = [np.nan, 60.0, 0.3, 0]
    for workers in (1, 3, 0):
        xycs, kept = prep(kps, w, h, workers)
        want = np.array([i for i in range(len(kps)) if port.in_margin(w, h, kps[i, 0], kps[i, 1])])
        assert np.array_equal(kept, want)
        assert np.array_equal(xycs[:, :2], kps[kept, :2])
        # same libm as the oracle: math.cos/sin are glibc's
        import math
        assert np.array_equal(xycs[:, 2], [math.cos(t) for t in kps[kept, 2]])
        assert np.array_equal(xycs[:, 3], [math.sin(t) for t in kps[kept, 2]])
    xy_only, kept2 = prep(kps[:, :2].copy(), w, h, 1)
    assert np.array_equal(kept2, kept) and np.all(xy_only[:, 2] == 1.0) and np.all(xy_only[:, 3] == 0.0)
    bad = kps[:10].copy()
    bad[3, 2] = np.inf
    with pytest.raises(RuntimeError):
        prep(bad, w, h, 1)


def test_filter_pass_matches_oracle(lib, port):
    from paper_1609_03986_b200.engine import Engine
    filt = Engine.filter_matches.__get__(type("E", (), {"lib": lib})())
    d = port.random_descriptors(77, 700, 64)
    probes, gallery = d[:300].copy(), d[300:].copy()
    gallery[9] = gallery[2]
    probes[4] = gallery[2]
    fwd = port.knn2_all(probes, gallery)
    rev = port.knn2_all(gallery, probes)[:, 0]
    for combo in range(8):
        kw = dict(ratio=0.85 if combo & 1 else None, max_distance=235 if combo & 4 else None)
        got = filt(fwd[:, 0], fwd[:, 1], fwd[:, 2], reverse_best=rev if combo & 2 else None, **kw)
        want = port.match(probes, gallery, cross_check=bool(combo & 2), **kw)
        assert np.array_equal(got, want)


def test_pattern_reader(ref=None):
    from paper_1609_03986_b200 import LatchError
    from paper_1609_03986_b200.pattern import default_pattern, format_pattern, parse_pattern
    pat = default_pattern()
    assert (pat.bit_count, pat.patch_size) == (512, 8) and pat.triplets.shape == (512, 6)
    w = pat.weights.reshape(8, 8)
    assert np.all(w[:7, :7] == 1.0) and np.all(w[7] == 0.0) and np.all(w[:, 7] == 0.0)
    text = format_pattern(pat)
    assert text.startswith("LATCHPAT v1 T=512 K=8\n") and text.count("\n") == 1 + 512 + 1 + 8
    assert parse_pattern(text).key() == pat.key()
    for name in ("t8k8", "t64k5w", "t16k12z", "t24k1"):
        text = (GOLDEN / f"pattern_{name}.latchpat").read_text()
        p = parse_pattern(text)
        T, K, trip, weights = oracle.parse_pattern_text(text)
        assert (p.bit_count, p.patch_size) == (T, K)
        assert np.array_equal(p.triplets, trip) and np.array_equal(p.weights, weights)
        assert parse_pattern(format_pattern(p)).key() == p.key()
    # error categories of src/pattern.cpp:68-131
    for text, code in [("", "BadHeader"), ("not a pattern", "BadHeader"),
                       ("LATCHPAT v1 T=12 K=8\n", "BadHeader"), ("LATCHPAT v1 T=8 K=0\n", "BadHeader"),
                       ("LATCHPAT v1 T=8 K=8\n1 2 3 4 5 6\n", "BadTripletCount"),
                       ("LATCHPAT v1 T=8 K=8\n" + "1 2 3 4 5 60\n" * 8, "CoordinateOutOfRange"),
                       ("LATCHPAT v1 T=8 K=8\n" + "1 2 3 4 3 4\n" * 8, "DegenerateTriplet"),
                       ("LATCHPAT v1 T=8 K=2\n" + "1 2 3 4 5 6\n" * 8 + "WEIGHTS\n0 0\n0 0\n", "BadHeader"),
                       ("LATCHPAT v1 T=8 K=2\n" + "1 2 3 4 5 6\n" * 8 + "WEIGHTS\n1 -1\n0 0\n", "BadHeader"),
                       ("LATCHPAT v1 T=8 K=8\n" + "1 2 3 4 5 6\n" * 9, "BadTripletCount")]:
        with pytest.raises(LatchError) as e:
            parse_pattern(text)
        assert e.value.code == code, text


def test_pattern_reader_agrees_with_reference(ref):
    from paper_1609_03986_b200.pattern import parse_pattern
    for name in ("t8k8", "t64k5w", "t16k12z", "t24k1"):
        text = (GOLDEN / f"pattern_{name}.latchpat").read_text()
        p = parse_pattern(text)
        T, K, trip, weights = ref.parse_pattern(text)
        assert (p.bit_count, p.patch_size) == (T, K)
        assert np.array_equal(p.triplets, trip) and np.array_equal(p.weights, weights)
    for bad in ("", "nope", "LATCHPAT v1 T=8 K=8\n1 2 3 4 5 6\n",
                "LATCHPAT v1 T=8 K=8\n" + "1 2 3 4 3 4\n" * 8):
        with pytest.raises(RuntimeError):
            ref.parse_pattern(bad)
        with pytest.raises(RuntimeError):
            parse_pattern(bad)


def test_argument_errors_need_no_device():
    import paper_1609_03986_b200 as lk
    with pytest.raises(ValueError):
        lk.describe(np.zeros(16), np.zeros((1, 2)))
    with pytest.raises(ValueError):
        lk.describe(np.zeros((100, 100)), np.zeros((1, 5)))
    with pytest.raises(RuntimeError):
        lk.describe(np.zeros((128, 128)), np.array([[64.0, 64.0]]), pattern="not a pattern")
    with pytest.raises(RuntimeError):
        lk.match(np.zeros((2, 64), np.uint8), np.zeros((0, 64), np.uint8))
    assert lk.match(np.zeros((0, 64), np.uint8), np.zeros((3, 64), np.uint8)).shape == (0, 4)
    with pytest.raises(RuntimeError):
        lk.hamming(np.zeros(64, np.uint8), np.zeros(32, np.uint8))
    assert (lk.descriptor_bits, lk.descriptor_bytes, lk.window_margin, lk.orientation_radius) == (512, 64, 46, 15)


def test_no_gpu_means_loud_failure_not_fallback():
    """On a box without CUDA the product must raise, never compute on the CPU."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1609_03986_b200 as lk
    from paper_1609_03986_b200 import ClatchDeviceError
    with pytest.raises(ClatchDeviceError):
        lk.describe(np.zeros((128, 128)), np.array([[64.0, 64.0]]))
    with pytest.raises(ClatchDeviceError):
        lk.match(np.zeros((2, 64), np.uint8), np.zeros((2, 64), np.uint8))
    with pytest.raises(ClatchDeviceError):
        lk.hamming(np.zeros(64, np.uint8), np.zeros(64, np.uint8))


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_1609_03986_b200"
    for path in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = path.read_text()
        assert "import oracle" not in text and "from oracle" not in text, path
        assert "latch_oracle" not in text and "liblatch_ref" not in text, path


def test_embedded_lane_placement_matches_the_builtin_table():
    """csrc/default_plan_f8.inc (generated by tools/gen_default_plan.py) is the filtered / pipelined
    kernels' lane placement of the built-in pattern: every slot must carry the window offsets
    (y * 65 + x) of one triplet, companions possibly swapped (bit 15), and the slots must be a
    permutation of the 512 triplets. A stale file would silently compute the wrong bits."""
    import re
    from pathlib import Path

    import numpy as np

    root = Path(__file__).resolve().parent.parent
    text = (root / "paper_1609_03986_b200" / "csrc" / "default_plan_f8.inc").read_text()
    stride = int(re.search(r"kDefaultPlanStride = (\d+)", text).group(1))
    rows = re.findall(r"\{(\d+), (\d+), (\d+), 0x([0-9a-f]{4})\}", text)
    assert len(rows) == 512 and stride == 65
    trip = np.load(root / "paper_1609_03986_b200" / "data" / "default_pattern.npz")["triplets"].astype(int)
    off = trip[:, 1::2] * stride + trip[:, 0::2]            # (512, 3): anchor, companion b, companion c
    seen = set()
    for a, b, c, w in rows:
        w = int(w, 16)
        t, swapped = w & 0x7FFF, w >> 15
        assert t not in seen
        seen.add(t)
        want = (off[t, 0], off[t, 2], off[t, 1]) if swapped else tuple(off[t])
        assert (int(a), int(b), int(c)) == tuple(int(v) for v in want), t
    assert seen == set(range(512))
    # conflict-freeness claim of the header: per group of 8 slots, residues mod 8 of each load
    slots = np.array([[int(a), int(b), int(c)] for a, b, c, _ in rows]).reshape(64, 8, 3) % 8
    worst = sum(np.bincount(slots[g, :, k], minlength=8).max() for g in range(64) for k in range(3)) / 192.0
    stated = float(re.search(r"kDefaultPlanDegree = ([0-9.]+)", text).group(1))
    assert abs(worst - stated) < 1e-6 and worst < 1.2


def test_ltch_container_round_trip_and_golden_bytes(tmp_path):
    """The LTCH container written from describe()'s arrays must be the reference's file byte for
    byte: tests/golden/golden_descriptors.bin is the regenerated fixture of acceptance.cpp:120-130
    (257 records, float32-narrowed keypoints). Errors keep the reference's categories."""
    import numpy as np
    import pytest

    from conftest import GOLDEN
    from paper_1609_03986_b200 import container as io

    blob = (GOLDEN / "golden_descriptors.bin").read_bytes()
    kps, desc = io.parse_descriptor_file(blob)
    assert kps.shape == (257, 4) and kps.dtype == np.float64 and desc.shape == (257, 64) and desc.dtype == np.uint8
    assert io.format_descriptor_file(kps, desc) == blob
    # from the float64 keypoints the detector produced: narrowing happens on write (static_cast<float>)
    kps64 = np.load(GOLDEN / "golden_keypoints_f64.npy")
    assert io.format_descriptor_file(kps64, desc) == blob
    io.save_descriptor_file(kps64, desc, tmp_path / "d.ltch")
    k2, d2 = io.load_descriptor_file(tmp_path / "d.ltch")
    assert np.array_equal(k2, kps) and np.array_equal(d2, desc)
    empty = io.format_descriptor_file(np.zeros((0, 4)), np.zeros((0, 64), np.uint8))
    assert empty == b"LTCH" + bytes([1, 0, 0, 0]) + bytes(12)          # count 0 -> descriptor bytes 0
    assert io.parse_descriptor_file(empty)[1].shape == (0, 0)
    for bad, what in ((b"LTCX" + blob[4:], "BadHeader"), (blob[:4] + bytes([2, 0, 0, 0]) + blob[8:], "BadHeader"),
                      (blob[:10], "Truncated"), (blob[:-1], "Truncated"), (blob[:20 + 80 * 3 + 7], "Truncated")):
        with pytest.raises(RuntimeError, match=what):
            io.parse_descriptor_file(bad)
    with pytest.raises(RuntimeError, match="Malformed"):
        io.load_descriptor_file(tmp_path / "missing.ltch")


def test_fp32_estimate_bound_never_decides_wrongly():
    """The filtered / pipelined extraction kernels take sign(d1 - d2) from fp32 sums over the
    truncated window only when |d1_f - d2_f| exceeds 2.2e-4 (sqrt d1_f + sqrt d2_f) + 3.3e-6 (d1_f + d2_f)
    + 3e-8. Restated here in numpy — cvt.rz truncation, one rounding per subtraction, one
    per fused accumulation, the bound in fp32 — against the reference's sequential fp64 chains, on
    windows built to sit on the decision boundary: whenever the estimate decides, it must agree."""
    import numpy as np

    rng = np.random.default_rng(160903986)

    def truncate32(v):                       # cvt.rz.f32.f64 for v >= 0
        f = v.astype(np.float32)
        over = f.astype(np.float64) > v
        f[over] = np.nextafter(f[over], np.float32(0))
        return f

    def exact_chain(a, b):                   # src/descriptor.cpp:61-75, 49 live terms, unfused
        d = np.zeros(len(a))
        for k in range(49):
            e = a[:, k] - b[:, k]
            d = d + e * e
        return d

    def fp32_chain(fa, fb):
        d = np.zeros(len(fa), np.float32)
        for k in range(49):
            e = fa[:, k] - fb[:, k]                                       # one rounding (fp32 subtraction)
            d = (e.astype(np.float64) * e.astype(np.float64) + d.astype(np.float64)).astype(np.float32)   # fused
        return d

    n = 40000
    cases = []
    base = rng.integers(0, 256, (n, 49)).astype(np.float64)
    frac = rng.random((n, 49))
    # 1. bilinear-like values of noise: everything far from a tie
    cases.append((rng.random((n, 49)) * 255, rng.random((n, 49)) * 255, rng.random((n, 49)) * 255))
    # 2. companions that differ from each other by perturbations from 1e-14 to 1e-1: the boundary region
    for scale in (1e-14, 1e-10, 1e-7, 3e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1):
        a = np.clip(base + frac, 0, 255)
        b = np.clip(a + rng.normal(0, 30, (n, 49)), 0, 255)
        c = np.clip(b + rng.normal(0, scale, (n, 49)), 0, 255)
        cases.append((a, b, c))
    # 3. flat and nearly flat footprints (the reference's bits are decided by rounding noise there)
    for scale in (0.0, 1e-15, 1e-13, 1e-9):
        level = rng.integers(0, 256, (n, 1)).astype(np.float64)
        mk = lambda: np.clip(level * (1 + rng.normal(0, 1, (n, 49)) * scale), 0, 255)   # noqa: E731
        cases.append((mk(), mk(), mk()))
    # 4. mirrored companions: d1 == d2 up to rounding, large sums
    a = rng.random((n, 49)) * 255
    delta = rng.normal(0, 40, (n, 49))
    cases.append((a, np.clip(a + delta, 0, 255), np.clip(a - delta, 0, 255)))

    decided_total = total = 0
    for a, b, c in cases:
        want = exact_chain(a, b) > exact_chain(a, c)
        fa, fb, fc = truncate32(a), truncate32(b), truncate32(c)
        assert np.all((a - fa.astype(np.float64) >= 0) & (a - fa.astype(np.float64) < 2.0 ** -16))
        d1, d2 = fp32_chain(fa, fb), fp32_chain(fa, fc)
        diff = d1 - d2
        bound = (np.float32(2.2e-4) * (np.sqrt(d1) + np.sqrt(d2)) + np.float32(3.3e-6) * (d1 + d2)
                 + np.float32(3.0e-8)).astype(np.float32)
        decided = np.abs(diff) > bound
        assert np.array_equal((diff > 0)[decided], want[decided])
        decided_total += int(decided.sum())
        total += len(decided)
    assert 0.15 < decided_total / total < 0.95       # the cases really straddle the boundary


def test_packed_plane_estimate_bound_never_decides_wrongly():
    """The default extraction kernel (extract_h16_kernel) estimates from 16-bit planes: a stored sample is an integer A
    with |A - 256 v| <= 0.66 (rounding 0.5 + fp32 / fixed-point resampling 0.16, csrc/clatch_extract.cu), differences
    of stored samples are exact in fp32, the sums are 49 fused fp32 accumulations, and a bit is taken from them only
    when |d1 - d2| > 19.1 (sqrt d1 + sqrt d2) + 3.3e-6 (d1 + d2) + 180. Restated in numpy against the reference's
    fp64 chains — with the stored samples pushed to the worst side the error budget allows (the first companion away
    from the anchor, the second towards it, and the other way round): whenever the estimate decides, it must agree."""
    import numpy as np

    rng = np.random.default_rng(16092)

    def exact_chain(a, b):                   # src/descriptor.cpp:61-75, 49 live terms, unfused
        d = np.zeros(len(a))
        for k in range(49):
            e = a[:, k] - b[:, k]
            d = d + e * e
        return d

    def stored(v, push, towards):
        """An integer within 0.66 of 256 v: nearest, or — where the budget allows — the neighbour further along `push`
        (+1 / -1 per element: away from or towards the anchor's stored value `towards`)."""
        x = 256.0 * v
        near = np.rint(x)
        direction = np.sign(near - towards) * push
        direction[direction == 0] = 1.0
        cand = np.where(direction > 0, np.floor(x) + 1.0, np.ceil(x) - 1.0)
        ok = np.abs(cand - x) <= 0.66
        return np.clip(np.where(ok, cand, near), 0, 65280)

    def fp32_chain(ia, ib):
        d = np.zeros(len(ia), np.float32)
        for k in range(49):
            e = (ia[:, k] - ib[:, k]).astype(np.float32)                  # exact: |e| <= 65280
            d = (e.astype(np.float64) * e.astype(np.float64) + d.astype(np.float64)).astype(np.float32)   # fused
        return d

    n = 30000
    cases = []
    base = rng.integers(0, 256, (n, 49)).astype(np.float64)
    frac = rng.random((n, 49))
    cases.append((rng.random((n, 49)) * 255, rng.random((n, 49)) * 255, rng.random((n, 49)) * 255))
    for scale in (1e-10, 1e-5, 1e-3, 3e-3, 1e-2, 3e-2, 1e-1, 0.3, 1.0):   # companions that differ by this much per pixel
        a = np.clip(base + frac, 0, 255)
        b = np.clip(a + rng.normal(0, 30, (n, 49)), 0, 255)
        c = np.clip(b + rng.normal(0, scale, (n, 49)), 0, 255)
        cases.append((a, b, c))
    for scale in (0.0, 1e-9, 1e-3, 1e-2):                                  # flat and nearly flat footprints
        level = rng.integers(0, 256, (n, 1)).astype(np.float64) + rng.random((n, 1))
        mk = lambda: np.clip(level + rng.normal(0, 1, (n, 49)) * scale, 0, 255)   # noqa: E731
        cases.append((mk(), mk(), mk()))
    a = rng.random((n, 49)) * 255                                          # mirrored companions: d1 == d2 up to rounding
    delta = rng.normal(0, 40, (n, 49))
    cases.append((a, np.clip(a + delta, 0, 255), np.clip(a - delta, 0, 255)))
    small = rng.random((n, 49)) * 0.02                                     # tiny sums: the constant term matters
    cases.append((small, rng.random((n, 49)) * 0.02, rng.random((n, 49)) * 0.02))

    decided_total = total = 0
    for a, b, c in cases:
        want = exact_chain(a, b) > exact_chain(a, c)
        ia = np.clip(np.rint(256.0 * a), 0, 65280)
        for push_b, push_c in ((1.0, -1.0), (-1.0, 1.0), (0.0, 0.0)):
            ib = stored(b, push_b, ia) if push_b else np.rint(256.0 * b)
            ic = stored(c, push_c, ia) if push_c else np.rint(256.0 * c)
            assert np.abs(ib - 256.0 * b).max() <= 0.66 and np.abs(ic - 256.0 * c).max() <= 0.66
            d1, d2 = fp32_chain(ia, ib), fp32_chain(ia, ic)
            diff = d1 - d2
            bound = (np.float32(19.1) * (np.sqrt(d1) + np.sqrt(d2)) + np.float32(3.3e-6) * (d1 + d2)
                     + np.float32(180.0)).astype(np.float32)
            decided = np.abs(diff) > bound
            assert np.array_equal((diff > 0)[decided], want[decided])
            decided_total += int(decided.sum())
            total += len(decided)
    assert 0.15 < decided_total / total < 0.95       # the cases really straddle the boundary


def test_take_keypoints_matches_numpy(lib):
    """clatch_take_keypoints: out[j] = kps[kept[j]] as (m, 4) rows, missing theta / score = 0
    (bindings/module.cpp:49-62), for every accepted column count and worker count."""
    import ctypes as C

    import numpy as np

    rng = np.random.default_rng(4)
    for cols in (2, 3, 4):
        for n in (1, 7, 5000, 40000):
            kps = rng.random((n, cols))
            kept = np.sort(rng.choice(n, size=max(1, n - n // 10), replace=False)).astype(np.int64)
            want = np.zeros((len(kept), 4))
            want[:, :cols] = kps[kept]
            for workers in (0, 1, 3):
                out = np.full((len(kept), 4), -1.0)
                rc = lib.clatch_take_keypoints(kps.ctypes.data_as(C.POINTER(C.c_double)), cols,
                                               kept.ctypes.data_as(C.POINTER(C.c_int64)), len(kept), workers,
                                               out.ctypes.data_as(C.POINTER(C.c_double)))
                assert rc == 0 and np.array_equal(out, want)
    assert lib.clatch_take_keypoints(None, 5, None, 0, 0, None) != 0          # bad column count


def test_image_rows_rule_copies_every_view_the_abi_cannot_take():
    """Engine._rows: the C ABI takes unit inner stride and a positive whole-element pitch >= width;
    flipped, transposed, broadcast and overlapping views are copied first (the reference accepts any
    array through c_style | forcecast, bindings/module.cpp:30)."""
    from paper_1609_03986_b200.engine import Engine
    for base in (np.arange(60, dtype=np.uint8).reshape(6, 10), np.arange(60, dtype=np.float64).reshape(6, 10)):
        for v in (base, base[::-1], base[:, ::-1], base.T, np.broadcast_to(base[0], (6, 10)), base[::2], base[:, 2:7],
                  base[::-1, ::-1][1:], base[:1]):
            a, pitch = Engine._rows(v)
            assert a.strides[1] == a.itemsize and pitch >= a.shape[1] and a.strides[0] == pitch * a.itemsize
            assert np.array_equal(a, v)
        a, pitch = Engine._rows(base[::2])
        assert np.shares_memory(a, base) and pitch == 20          # a plain row-skipping view needs no copy


def test_bench_reference_arm_and_workload_strings():
    """`bench.py --impl reference` prints one JSON line whose config.workload is the string our arm
    prints for the same configuration (both come from oracle/workloads.py)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--workload", "cfg1", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    from oracle import workloads
    assert line["impl"] == "reference" and line["config"]["workload"] == workloads.DESCRIPTIONS["cfg1"]
    assert line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1 and line["e2e"]["h2d_bytes_per_step"] == 0
    src = (root / "bench.py").read_text()
    assert src.count("DESCRIPTIONS[") >= 6 and "u8-valued noise image" not in src   # one source for both arms


def test_cfg4_workload_has_the_planted_structure():
    """oracle/workloads.cfg4_sets at a small size: planted copies are exact copies of FINAL train rows and
    duplicated train rows exist (the tie cases of proj/tests/acceptance.cpp:170-173)."""
    from oracle import workloads
    q, t, (dup_q, src_t) = workloads.cfg4_sets(rows=20_000)
    assert q.shape == t.shape == (20_000, 64) and len(dup_q) == 200
    assert np.array_equal(q[dup_q], t[src_t])
    _, counts = np.unique(t, axis=0, return_counts=True)
    assert (counts > 1).sum() >= 15
    res = workloads.knn2_rows_threaded(q[dup_q[:8]], t)
    assert np.all(res[:, 1] == 0) and np.all(res[:, 0] <= src_t[:8])
    rows = workloads.match_threaded(q[:300], t[:500], ratio=0.8, cross_check=True)
    import oracle
    assert np.array_equal(rows, oracle.port().match(q[:300], t[:500], ratio=0.8, cross_check=True))
