#!/usr/bin/env python
"""GPU probe for the tcgen05 matcher: raw accumulator tile vs 512 - 2*hamming, then top-2 vs
the oracle on growing shapes. Run under `timeout`; prints enough to localise a layout bug."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle                                     # noqa: E402
from paper_1609_03986_b200 import _lib            # noqa: E402
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

port = oracle.port()
eng = get_engine()
lib = eng.lib


def tile(q, t):
    out = np.zeros((128, 256), np.int32)
    res = np.zeros((3, len(q)), np.int32)
    p = lambda a, ty: a.ctypes.data_as(ty)
    _lib.check(lib.clatch_debug_tc_tile(eng.ctx, p(q, _lib.u8p), len(q), p(t, _lib.u8p), len(t), p(out, _lib.i32p),
                                        p(res[0], _lib.i32p), p(res[1], _lib.i32p), p(res[2], _lib.i32p)))
    return out, res


d = port.random_descriptors(1, 128 + 256, 64)
q, t = d[:128].copy(), d[128:].copy()
got, res = tile(q, t)
ham = np.unpackbits(q[:, None, :] ^ t[None, :, :], axis=2).sum(2).astype(np.int32)
want = 512 - 2 * ham
ok = np.array_equal(got, want)
print("raw tile exact:", ok, flush=True)
if not ok:
    bad = np.argwhere(got != want)
    print("mismatches:", len(bad), "of", got.size, "first:", bad[:8].tolist())
    print("got[0,:8]", got[0, :8].tolist(), "want[0,:8]", want[0, :8].tolist())
    print("got[:8,0]", got[:8, 0].tolist(), "want[:8,0]", want[:8, 0].tolist())
    print("rows fully right:", int((got == want).all(1).sum()), "cols fully right:", int((got == want).all(0).sum()))
    # is it a permutation problem? compare sorted rows
    print("row multisets equal:", int(sum(np.array_equal(np.sort(a), np.sort(b)) for a, b in zip(got, want))))
    print("transposed match:", np.array_equal(got[:128, :128], want[:128, :128].T))
print("top2 exact:", np.array_equal(res.T, port.knn2_all(q, t)), flush=True)

eng.set_option("match_variant", 3)
for nq, nt in [(1, 1), (100, 300), (128, 512), (129, 257), (1000, 5000), (3000, 20000)]:
    dd = port.random_descriptors(50 + nq + nt, nq + nt, 64)
    qq, tt = dd[:nq].copy(), dd[nq:].copy()
    if nt > 2:
        tt[nt - 1] = tt[0]
        qq[0] = tt[0]
    bi, bd, sd = eng.match_top2(qq, tt)
    w = port.knn2_all(qq, tt)
    okk = np.array_equal(np.stack([bi, bd, sd], 1), w)
    print(f"Q={nq} N={nt}: exact={okk}", flush=True)
    if not okk:
        g = np.stack([bi, bd, sd], 1)
        bad = np.argwhere((g != w).any(1)).ravel()
        print("  bad rows", len(bad), bad[:10].tolist(), "got", g[bad[:3]].tolist(), "want", w[bad[:3]].tolist())
print("probe done")
