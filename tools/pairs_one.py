#!/usr/bin/env python
"""All pairs of `n` resident random descriptor sets of `rows` rows (cfg5 shape) in one call, timed: pairs_one.py n rows [reps]."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

n, rows = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
eng = get_engine()
rng = np.random.default_rng(0)
sets = [eng.create_set(rng.integers(0, 256, (rows, 64), dtype=np.uint8)) for _ in range(n)]
pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
eng.match_set_pairs(sets, pairs, ratio=0.8, cross_check=True)
t0 = time.perf_counter()
for _ in range(reps):
    eng.match_set_pairs(sets, pairs, ratio=0.8, cross_check=True)
dt = (time.perf_counter() - t0) / reps
print({"sets": n, "rows": rows, "pairs": len(pairs), "ms": dt * 1e3, "pairs_per_s": len(pairs) / dt,
       "compares_per_s": 2 * len(pairs) * rows * rows / dt})
