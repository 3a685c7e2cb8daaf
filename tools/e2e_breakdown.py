#!/usr/bin/env python
"""Where does the host-API step time go? Times the pieces of describe()+match() on cfg2."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench                                        # noqa: E402
import paper_1609_03986_b200 as lk                  # noqa: E402

img, kps = bench.synth_inputs("cfg2")
eng = lk.get_engine()
eng.set_pattern(None)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def timeit(fn, reps=30):
    for _ in range(5):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return (time.perf_counter() - t0) / reps * 1e3, out


img64, img8, k = pinned(img.astype(np.float64)), pinned(img), pinned(kps)
h, w = img.shape
ms, (xycs, kept) = timeit(lambda: eng.prepare_keypoints(k, w, h))
print(f"prepare_keypoints            {ms:.3f} ms")
for workers in (1, 2, 4, 8, 0):
    ms, _ = timeit(lambda: eng.prepare_keypoints(k, w, h, workers))
    print(f"prepare_keypoints workers={workers} {ms:.3f} ms")
ms, desc = timeit(lambda: eng.extract(img8, xycs))
print(f"extract u8 (H2D+kernel+D2H)  {ms:.3f} ms")
ms, desc = timeit(lambda: eng.extract(img64, xycs))
print(f"extract f64                  {ms:.3f} ms")
ms, _ = timeit(lambda: eng.describe_all(img8, k))
print(f"describe_all u8              {ms:.3f} ms")
ms, _ = timeit(lambda: eng.describe_all(img64, k))
print(f"describe_all f64             {ms:.3f} ms")
ms, _ = timeit(lambda: lk.describe(img8, k))
print(f"lk.describe u8               {ms:.3f} ms")
ms, _ = timeit(lambda: lk.describe(img64, k))
print(f"lk.describe f64              {ms:.3f} ms")
eng.set_option("host_promote", 1)
ms, _ = timeit(lambda: lk.describe(img64, k))
print(f"lk.describe f64, host_promote=1 (u8 conversion on the host workers, 2 MB upload) {ms:.3f} ms")
eng.set_option("host_promote", 0)
pageable = img.astype(np.float64)
ms, _ = timeit(lambda: lk.describe(pageable, k))
print(f"lk.describe f64 pageable image {ms:.3f} ms")
_, desc = lk.describe(img8, k)                      # page-locked result array, as the API returns it
ms, _ = timeit(lambda: eng.match_top2(desc, desc))
print(f"match_top2 host              {ms:.3f} ms")
ms, _ = timeit(lambda: eng.match_brute_force(desc, desc))
print(f"match_brute_force host       {ms:.3f} ms")
ms, _ = timeit(lambda: lk.match(desc, desc))
print(f"lk.match                     {ms:.3f} ms")
dpage = desc.copy()
ms, _ = timeit(lambda: lk.match(dpage, dpage))
print(f"lk.match pageable arrays     {ms:.3f} ms")
ms, _ = timeit(lambda: lk.match(desc, desc, ratio=0.8, cross_check=True))
print(f"lk.match ratio+cross         {ms:.3f} ms")
d_img = torch.from_numpy(img).cuda()
d_x = torch.from_numpy(xycs).cuda()
d_desc = eng.extract_device(d_img, d_x)
def dev():
    eng.extract_device(d_img, d_x, out=d_desc); eng.match_top2_device(d_desc, d_desc); torch.cuda.synchronize()
ms, _ = timeit(dev)
print(f"device-resident step (wall)  {ms:.3f} ms")
t = torch.from_numpy(img64)
ms, _ = timeit(lambda: (t.cuda(non_blocking=True), torch.cuda.synchronize()))
print(f"torch H2D 16.6 MB pinned     {ms:.3f} ms")
