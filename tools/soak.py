#!/usr/bin/env python
"""Randomised soak of the extraction and matching paths against the oracle: random image sizes and
kinds, keypoint counts, kernel variants, host / device / batch / banded entry points.

    python tools/soak.py [seconds]        (default 120)
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle                                   # noqa: E402
import paper_1609_03986_b200 as lk              # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
port = oracle.port()
eng = lk.get_engine()
rng = np.random.default_rng(20260917)
t_end = time.time() + budget
cases = {"describe": 0, "device": 0, "batch": 0, "banded": 0, "match": 0, "pairs": 0}


def image(kind, w, h):
    if kind == "noise":
        return rng.integers(0, 256, (h, w)).astype(np.uint8)
    if kind == "flatish":
        return (rng.integers(0, 4, (h // 32 + 1, w // 32 + 1)) * 64).astype(np.uint8).repeat(32, 0).repeat(32, 1)[:h, :w]
    if kind == "lsb":
        return (200 + rng.integers(0, 2, (h, w))).astype(np.uint8)
    yy, xx = np.mgrid[0:h, 0:w]
    return ((np.sin(xx / 9.0) * np.cos(yy / 7.0) * 100 + 128) + rng.integers(-3, 4, (h, w))).clip(0, 255).astype(np.uint8)


it = 0
while time.time() < t_end:
    it += 1
    w, h = int(rng.integers(93, 700)), int(rng.integers(93, 500))
    n = int(rng.choice([1, 3, 4, 5, 17, 128, 400, 1500]))
    kind = str(rng.choice(["noise", "flatish", "lsb", "smooth"]))
    img = image(kind, w, h)
    kps = np.column_stack([rng.uniform(40, w - 40, n), rng.uniform(40, h - 40, n), rng.uniform(-7, 7, n), rng.random(n)])
    if rng.random() < 0.3:
        kps[:, :2] = np.floor(kps[:, :2]) + rng.choice([0.0, 0.5])
    variant = int(rng.choice([0, 1, 2, 3, 4, 5, 5, 5, 6, 6]))    # weighted towards the packed-plane kernels (5 = default)
    eng.set_option("extract_variant", variant)
    as_f64 = rng.random() < 0.4
    src = img.astype(np.float64) + (rng.random(img.shape) * 0.3 if rng.random() < 0.3 and as_f64 else 0.0) if as_f64 else img
    if as_f64 and rng.random() < 0.3:                                    # other value ranges: the float64 route of the default kernel
        scale = 10.0 ** float(rng.uniform(-60, 60))
        src = (src + rng.random(img.shape) * 0.7) * scale + float(rng.choice([0.0, 37.25, -1e3, 3e5])) * scale
    if as_f64:
        eng.set_option("host_promote", int(rng.integers(0, 3)))          # pageable rule / always / never
        if rng.random() < 0.15:                                          # non-finite pixels: the literal (w*e)*e kernel
            src = src.copy()
            src[int(rng.integers(0, h)), int(rng.integers(0, w))] = [np.nan, np.inf, -np.inf, 1e308][int(rng.integers(0, 4))]
    with np.errstate(all="ignore"):
        kept_idx, want = port.describe_all(np.asarray(src, np.float64), kps)
    kept, desc = lk.describe(src, kps)
    assert np.array_equal(kept, kps[kept_idx]) and np.array_equal(desc, want), ("describe", it, w, h, n, kind, variant, as_f64)
    cases["describe"] += 1
    if len(kept_idx) and src.dtype == np.uint8:
        xycs, _ = eng.prepare_keypoints(kps, w, h)
        got = eng.extract_device(torch.from_numpy(src).cuda(), torch.from_numpy(xycs).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), want), ("device", it, w, h, n, kind, variant)
        cases["device"] += 1
    if it % 5 == 0:
        imgs = [image(str(rng.choice(["noise", "smooth"])), w + 7 * j, h + 3 * j) for j in range(3)]
        kl = [np.column_stack([rng.uniform(46, im.shape[1] - 47, 60 + j), rng.uniform(46, im.shape[0] - 47, 60 + j),
                               rng.uniform(-3, 3, 60 + j), np.zeros(60 + j)]) for j, im in enumerate(imgs)]
        for (k2, d2), im, k in zip(lk.describe_batch(imgs, kl), imgs, kl):
            assert np.array_equal(d2, port.describe_all(im.astype(np.float64), k)[1]), ("batch", it, variant)
        cases["batch"] += 1
    if it % 9 == 0:                                   # banded float64 upload: needs a big frame and >= 4096 keypoints
        eng.set_option("extract_variant", 5)
        W, H, N = 1100 + int(rng.integers(0, 200)), 800 + int(rng.integers(0, 100)), 4200
        big = image("noise", W, H).astype(np.float64)
        if rng.random() < 0.5:
            big[int(rng.integers(0, H)), int(rng.integers(0, W))] += 0.5
        k = np.column_stack([rng.uniform(40, W - 40, N), rng.uniform(40, H - 40, N), rng.uniform(-4, 4, N), np.zeros(N)])
        eng.set_option("upload_bands", int(rng.integers(0, 5)))
        assert np.array_equal(lk.describe(big, k)[1], port.describe_all(big, k)[1]), ("banded", it)
        eng.set_option("upload_bands", 0)
        cases["banded"] += 1
    # matching
    q_n, t_n = int(rng.choice([1, 2, 127, 129, 600, 3000, 9000])), int(rng.choice([1, 2, 239, 241, 255, 257, 1000, 5000, 12000]))
    q, t = port.random_descriptors(it, q_n), port.random_descriptors(it + 100000, t_n)
    for j in range(0, q_n, 5):
        q[j] = t[int(rng.integers(0, t_n))]
    eng.set_option("match_streamk", int(rng.integers(0, 2)))
    eng.set_option("match_variant", int(rng.choice([3, 4, 4])))          # int8 / e2m1 operands on the tensor cores
    eng.set_option("match_pairs", int(rng.integers(0, 2)))               # CTA pairs sharing the train stream or not
    kw = [{}, {"ratio": 0.8}, {"cross_check": True}, {"ratio": 0.9, "cross_check": True, "max_distance": 230}][int(rng.integers(0, 4))]
    assert np.array_equal(lk.match(q, t, **kw), port.match(q, t, **kw)), ("match", it, q_n, t_n, kw)
    cases["match"] += 1
    if it % 7 == 0:
        sets_raw = [port.random_descriptors(it * 10 + j, int(rng.choice([1, 130, 500]))) for j in range(4)]
        sets_raw[2][0] = sets_raw[0][0]
        sets = [eng.create_set(s) for s in sets_raw]
        pairs = [(a, b) for a in range(4) for b in range(4) if a != b]
        eng.set_option("pairs_filter_on_device", int(rng.integers(0, 2)))
        for (a, b), got in zip(pairs, eng.match_set_pairs(sets, pairs, **kw)):
            assert np.array_equal(got, port.match(sets_raw[a], sets_raw[b], **kw)), ("pairs", it, a, b, kw)
        eng.set_option("pairs_filter_on_device", 1)
        for s in sets:
            s.close()
        cases["pairs"] += 1
eng.set_option("extract_variant", 5)
eng.set_option("match_streamk", 1)
eng.set_option("match_variant", 4)
eng.set_option("match_pairs", 1)
eng.set_option("host_promote", 0)
print(f"soak ok: {it} iterations in {budget:.0f} s; cases {cases}")
