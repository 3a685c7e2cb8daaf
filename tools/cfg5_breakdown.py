#!/usr/bin/env python
"""Where the cfg5 end-to-end time goes (256 images x 8000 keypoints, all pairs): stage by stage, host clock."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import workloads as W                       # noqa: E402
import paper_1609_03986_b200 as lk                      # noqa: E402
from paper_1609_03986_b200 import sharded               # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
imgs, kps = W.images_and_keypoints("cfg5", range(n))
dev = torch.device("cuda", 0)
eng = lk.get_engine()
for kind, arr in (("u8", imgs), ("f64", [a.astype(np.float64) for a in imgs])):
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        local = sharded.extract_images_sharded(arr, kps)
        t1 = time.perf_counter()
        sets = sharded.all_gather_descriptor_sets({i: v[1] for i, v in local.items()}, n, device=dev)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        res = sharded.create_resident_sets(sets, n)
        eng.synchronize()
        t3 = time.perf_counter()
        out = sharded.match_all_pairs_resident(sets, ratio=W.RATIO, cross_check=True, num_images=n, resident=res)
        t4 = time.perf_counter()
        for s in res.values():
            s.close()
        t5 = time.perf_counter()
        print(f"{kind} rep {rep}: extract {1e3 * (t1 - t0):.1f} ms, gather {1e3 * (t2 - t1):.1f} ms, create sets {1e3 * (t3 - t2):.1f} ms, "
              f"match {1e3 * (t4 - t3):.1f} ms, close {1e3 * (t5 - t4):.1f} ms, total {1e3 * (t5 - t0):.1f} ms "
              f"({n * (n - 1) // 2 / (t5 - t0):.0f} pairs/s)")
