"""TEST INFRASTRUCTURE — CPU checkers for the CLATCH hot paths. Not the product.

Two checkers, both reached through ctypes:

* ``port``  — ``oracle/liblatch_oracle.so``, the plain-C restatement in
  ``oracle/latch_oracle.c`` (travels everywhere; built by ``make -C oracle``).
* ``ref``   — ``oracle/_ref/liblatch_ref.so``, the UNMODIFIED reference compiled
  from ``/root/reference/proj`` by ``oracle/build_ref.sh`` (git-ignored; shipped
  to the GPU box as a prebuilt artefact). ``None`` when it has not been built.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product
(``paper_1609_03986_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liblatch_oracle.so"
REF_SO = HERE / "_ref" / "liblatch_ref.so"
PATTERN_FILE = HERE.parent / "paper_1609_03986_b200" / "data" / "default_pattern.npz"

_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build_port() -> None:
    """Compile the C restatement if it is missing or stale."""
    src = HERE / "latch_oracle.c"
    if not PORT_SO.exists() or PORT_SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "liblatch_oracle.so"], check=True,
                       stdout=subprocess.DEVNULL)


def parse_pattern_text(text: str):
    """Minimal reader of the LATCHPAT v1 text (proj/src/pattern.cpp:68-131) for the
    checker's own use: returns (T, K, triplets int32 (T,6), weights f64 (K*K,))."""
    lines = [ln for ln in text.split("\n")]
    head = lines[0].split()
    T = int(head[2].split("=")[1])
    K = int(head[3].split("=")[1])
    trip = []
    i = 1
    weights = None
    while i < len(lines):
        ln = lines[i]
        i += 1
        if not ln:
            continue
        if ln == "WEIGHTS":
            vals = []
            for _ in range(K):
                vals.extend(float(v) for v in lines[i].split()[:K])
                i += 1
            weights = np.array(vals, dtype=np.float64)
            break
        trip.append([int(v) for v in ln.split()[:6]])
    if weights is None:
        weights = np.ones(K * K, dtype=np.float64)
    return T, K, np.array(trip, dtype=np.int32).reshape(T, 6), weights


def default_pattern():
    """(T, K, triplets int32 (T,6), weights f64 (K*K,)) of the shipped table (data file only;
    the checker never imports the product package)."""
    d = np.load(PATTERN_FILE)
    return (int(d["bit_count"]), int(d["patch_size"]), d["triplets"].astype(np.int32),
            d["weights"].astype(np.float64))


class Port:
    """ctypes face of oracle/latch_oracle.c."""

    def __init__(self):
        build_port()
        self.lib = L = C.CDLL(str(PORT_SO))
        L.oracle_rng_next.argtypes = [C.c_uint64, C.c_size_t, _u64p]
        L.oracle_rng_units.argtypes = [C.c_uint64, C.c_size_t, _f64p]
        L.oracle_random_image.argtypes = [C.c_uint64, C.c_int, C.c_int, _f64p]
        L.oracle_random_image_u8.argtypes = [C.c_uint64, C.c_int, C.c_int, _u8p]
        L.oracle_structured_image.argtypes = [C.c_uint64, C.c_int, C.c_int, _f64p]
        L.oracle_random_descriptors.argtypes = [C.c_uint64, C.c_size_t, C.c_int, _u8p]
        L.oracle_random_keypoints.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_size_t, _f64p]
        L.oracle_in_margin.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.oracle_in_margin.restype = C.c_int
        L.oracle_sample_bilinear.argtypes = [_f64p, C.c_int, C.c_int, C.c_double, C.c_double]
        L.oracle_sample_bilinear.restype = C.c_double
        L.oracle_extract_window.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _f64p]
        L.oracle_extract_window.restype = C.c_int
        L.oracle_triplet_bit.argtypes = [_f64p, _i32p, C.c_int, _f64p]
        L.oracle_triplet_bit.restype = C.c_int
        L.oracle_describe.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _i32p, C.c_int, C.c_int,
                                      _f64p, _u8p]
        L.oracle_describe.restype = C.c_int
        L.oracle_describe_all.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_size_t, _i32p,
                                          C.c_int, C.c_int, _f64p, _i64p, _u8p]
        L.oracle_describe_all.restype = C.c_size_t
        L.oracle_hamming.argtypes = [_u8p, _u8p, C.c_size_t]
        L.oracle_hamming.restype = C.c_int
        L.oracle_knn2.argtypes = [_u8p, _u8p, C.c_size_t, C.c_int, _i32p]
        L.oracle_knn2_range.argtypes = [_u8p, C.c_size_t, C.c_size_t, _u8p, C.c_size_t, C.c_int,
                                        _i32p]
        L.oracle_filter_matches.argtypes = [_i32p, C.c_size_t, C.c_int, C.c_double, C.c_int,
                                            C.c_int, _i32p, _i32p]
        L.oracle_filter_matches.restype = C.c_size_t
        L.oracle_match.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.c_int, C.c_int,
                                   C.c_double, C.c_int, C.c_int, C.c_int, _i32p]
        L.oracle_match.restype = C.c_size_t
        L.oracle_triplet_bits.argtypes = [_f64p, C.c_size_t, _i32p, C.c_size_t, C.c_int, _f64p, _u8p, C.c_size_t]
        L.oracle_fast_detect.argtypes = [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, _f64p, C.c_size_t]
        L.oracle_fast_detect.restype = C.c_size_t
        L.oracle_detect_and_orient.argtypes = [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _f64p,
                                               C.c_size_t]
        L.oracle_detect_and_orient.restype = C.c_size_t

    # ---- generators ----
    def rng_next(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.oracle_rng_next(seed, n, _p(out, _u64p))
        return out

    def rng_units(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.oracle_rng_units(seed, n, _p(out, _f64p))
        return out

    def random_image(self, seed, w, h):
        out = np.empty((h, w), np.float64)
        self.lib.oracle_random_image(seed, w, h, _p(out, _f64p))
        return out

    def random_image_u8(self, seed, w, h):
        out = np.empty((h, w), np.uint8)
        self.lib.oracle_random_image_u8(seed, w, h, _p(out, _u8p))
        return out

    def structured_image(self, seed, w, h):
        out = np.empty((h, w), np.float64)
        self.lib.oracle_structured_image(seed, w, h, _p(out, _f64p))
        return out

    def random_descriptors(self, seed, n, nbytes=64):
        out = np.empty((n, nbytes), np.uint8)
        self.lib.oracle_random_descriptors(seed, n, nbytes, _p(out, _u8p))
        return out

    def random_keypoints(self, seed, w, h, n):
        out = np.empty((n, 4), np.float64)
        self.lib.oracle_random_keypoints(seed, w, h, n, _p(out, _f64p))
        return out

    # ---- extraction ----
    def in_margin(self, w, h, x, y):
        return bool(self.lib.oracle_in_margin(w, h, x, y))

    def extract_window(self, image, kp):
        image = np.ascontiguousarray(image, np.float64)
        kp = np.ascontiguousarray(kp, np.float64)
        win = np.empty(4096, np.float64)
        h, w = image.shape
        if self.lib.oracle_extract_window(_p(image, _f64p), w, h, _p(kp, _f64p), _p(win, _f64p)):
            raise RuntimeError("TooCloseToBorder")
        return win

    def triplet_bit(self, win, trip, K, weights):
        win = np.ascontiguousarray(win, np.float64)
        trip = np.ascontiguousarray(trip, np.int32)
        weights = np.ascontiguousarray(weights, np.float64)
        return bool(self.lib.oracle_triplet_bit(_p(win, _f64p), _p(trip, _i32p), K,
                                                _p(weights, _f64p)))

    def describe(self, image, kp, pattern=None):
        T, K, trip, weights = pattern or default_pattern()
        image = np.ascontiguousarray(image, np.float64)
        kp = np.ascontiguousarray(kp, np.float64)
        out = np.zeros(T // 8, np.uint8)
        h, w = image.shape
        if self.lib.oracle_describe(_p(image, _f64p), w, h, _p(kp, _f64p), _p(trip, _i32p), T, K,
                                    _p(weights, _f64p), _p(out, _u8p)):
            raise RuntimeError("TooCloseToBorder")
        return out

    def describe_all(self, image, kps, pattern=None):
        """-> (kept input indices int64 (M,), descriptors uint8 (M, T/8))."""
        T, K, trip, weights = pattern or default_pattern()
        image = np.ascontiguousarray(image, np.float64)
        kps = np.ascontiguousarray(kps, np.float64)
        n = len(kps)
        h, w = image.shape
        kept = np.empty(n, np.int64)
        desc = np.zeros((n, T // 8), np.uint8)
        m = self.lib.oracle_describe_all(_p(image, _f64p), w, h, _p(kps, _f64p), n,
                                         _p(trip, _i32p), T, K, _p(weights, _f64p),
                                         _p(kept, _i64p), _p(desc, _u8p))
        return kept[:m].copy(), desc[:m].copy()

    # ---- trainer scoring ----
    def triplet_bits(self, windows, candidates, K, weights):
        """-> uint8 (C, ceil(n/8)): bit i of row c = triplet_bit(window i, candidate c)."""
        windows = np.ascontiguousarray(windows, np.float64).reshape(-1, 4096)
        cand = np.ascontiguousarray(candidates, np.int32).reshape(-1, 6)
        weights = np.ascontiguousarray(weights, np.float64)
        n, c = len(windows), len(cand)
        row = (n + 7) // 8
        out = np.zeros((c, row), np.uint8)
        self.lib.oracle_triplet_bits(_p(windows, _f64p), n, _p(cand, _i32p), c, K, _p(weights, _f64p),
                                     _p(out, _u8p), row)
        return out

    # ---- detection ----
    def detect(self, image, threshold=20.0, nms=True, orient=True, radius=15):
        """fast_detect / detect_and_orient -> (N, 4) float64 [x, y, theta, score]."""
        image = np.ascontiguousarray(image, np.float64)
        h, w = image.shape
        cap = max(w * h, 1)
        out = np.empty((cap, 4), np.float64)
        if orient:
            n = self.lib.oracle_detect_and_orient(_p(image, _f64p), w, h, threshold, int(nms), radius,
                                                  _p(out, _f64p), cap)
        else:
            n = self.lib.oracle_fast_detect(_p(image, _f64p), w, h, threshold, int(nms), _p(out, _f64p), cap)
        if n == C.c_size_t(-1).value:
            raise RuntimeError("ImageTooSmall")
        return out[:n].copy()

    # ---- matching ----
    def hamming(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        assert a.shape == b.shape
        return int(self.lib.oracle_hamming(_p(a, _u8p), _p(b, _u8p), a.size))

    def knn2(self, probe, gallery):
        probe = np.ascontiguousarray(probe, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        out = np.empty(3, np.int32)
        self.lib.oracle_knn2(_p(probe, _u8p), _p(gallery, _u8p), len(gallery), gallery.shape[1],
                             _p(out, _i32p))
        return tuple(int(v) for v in out)

    def knn2_all(self, probes, gallery, begin=0, end=None):
        """-> int32 (Q,3) [best_index, best_distance, second_distance]; only rows
        [begin, end) are filled."""
        probes = np.ascontiguousarray(probes, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        q = len(probes)
        end = q if end is None else end
        out = np.zeros((q, 3), np.int32)
        self.lib.oracle_knn2_range(_p(probes, _u8p), begin, end, _p(gallery, _u8p), len(gallery),
                                   gallery.shape[1], _p(out, _i32p))
        return out

    def match(self, probes, gallery, ratio=None, cross_check=False, max_distance=None):
        probes = np.ascontiguousarray(probes, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        q, n = len(probes), len(gallery)
        nbytes = gallery.shape[1] if gallery.ndim == 2 else probes.shape[1]
        out = np.empty((max(q, 1), 4), np.int32)
        m = self.lib.oracle_match(_p(probes, _u8p), q, _p(gallery, _u8p), n, nbytes,
                                  int(ratio is not None), float(ratio or 0.0), int(cross_check),
                                  int(max_distance is not None), int(max_distance or 0),
                                  _p(out, _i32p))
        if m == C.c_size_t(-1).value:
            raise RuntimeError("EmptyGallery")
        return out[:m].copy()


class Ref:
    """ctypes face of the unmodified reference (oracle/_ref/liblatch_ref.so)."""

    def __init__(self):
        self.lib = L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_units.argtypes = [C.c_uint64, C.c_size_t, _f64p]
        L.ref_rng_next.argtypes = [C.c_uint64, C.c_size_t, _u64p]
        L.ref_random_image.argtypes = [C.c_uint64, C.c_int, C.c_int, _f64p]
        L.ref_structured_image.argtypes = [C.c_uint64, C.c_int, C.c_int, _f64p]
        L.ref_random_descriptors.argtypes = [C.c_uint64, C.c_size_t, C.c_int, _u8p]
        L.ref_default_pattern_text.argtypes = [C.c_char_p, C.c_size_t]
        L.ref_default_pattern_text.restype = C.c_size_t
        L.ref_parse_pattern.argtypes = [C.c_char_p, _i32p, _i32p, _i32p, C.c_size_t, _f64p,
                                        C.c_size_t]
        L.ref_detect_and_orient.argtypes = [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, _f64p,
                                            C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_triplet_bits.argtypes = [_f64p, C.c_size_t, _i32p, C.c_size_t, C.c_int, _f64p, _u8p, C.c_size_t]
        L.ref_sample_candidates.argtypes = [C.c_size_t, C.c_int, C.c_uint64, _i32p]
        L.ref_fast_detect.argtypes = [_f64p, C.c_int, C.c_int, C.c_double, C.c_int, _f64p,
                                      C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_load_pgm.argtypes = [C.c_char_p, _f64p, C.c_size_t, _i32p, _i32p]
        L.ref_keypoint_in_margin.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
        L.ref_extract_window.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _f64p]
        L.ref_oracle_window.argtypes = [_f64p, C.c_int, C.c_int, _f64p, _f64p]
        L.ref_triplet_bit.argtypes = [_f64p, _i32p, C.c_int, _f64p]
        L.ref_describe.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_char_p, _u8p]
        L.ref_oracle_describe.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_char_p, _u8p]
        L.ref_describe_all.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_size_t, C.c_char_p,
                                       C.c_int, _i64p, _u8p, C.POINTER(C.c_size_t)]
        L.ref_describe_all_file.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_size_t,
                                            C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_hamming.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, _i32p]
        L.ref_knn2.argtypes = [_u8p, _u8p, C.c_size_t, C.c_int, _i32p]
        L.ref_knn2_all.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.c_int, _i32p]
        L.ref_match.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.c_int, C.c_int, C.c_double,
                                C.c_int, C.c_int, C.c_int, C.c_int, _i32p,
                                C.POINTER(C.c_size_t)]
        L.ref_oracle_match.argtypes = [_u8p, C.c_size_t, _u8p, C.c_size_t, C.c_int, C.c_int,
                                       C.c_double, C.c_int, C.c_int, C.c_int, _i32p,
                                       C.POINTER(C.c_size_t)]
        L.ref_bench_create.argtypes = [_f64p, C.c_int, C.c_int, _f64p, C.c_size_t]
        L.ref_bench_create.restype = C.c_void_p
        L.ref_bench_destroy.argtypes = [C.c_void_p]
        L.ref_bench_describe.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
        L.ref_bench_describe.restype = C.c_size_t
        L.ref_bench_set_gallery.argtypes = [C.c_void_p, _u8p, C.c_size_t, C.c_int]
        L.ref_bench_gallery_from_probes.argtypes = [C.c_void_p]
        L.ref_bench_set_probes.argtypes = [C.c_void_p, _u8p, C.c_size_t, C.c_int]
        L.ref_bench_match.argtypes = [C.c_void_p, C.c_size_t, C.c_int, _u64p]
        L.ref_bench_match.restype = C.c_size_t

    def _check(self, rc):
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def rng_next(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng_next(seed, n, _p(out, _u64p))
        return out

    def rng_units(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.ref_rng_units(seed, n, _p(out, _f64p))
        return out

    def random_image(self, seed, w, h):
        out = np.empty((h, w), np.float64)
        self.lib.ref_random_image(seed, w, h, _p(out, _f64p))
        return out

    def structured_image(self, seed, w, h):
        out = np.empty((h, w), np.float64)
        self.lib.ref_structured_image(seed, w, h, _p(out, _f64p))
        return out

    def random_descriptors(self, seed, n, nbytes=64):
        out = np.empty((n, nbytes), np.uint8)
        self.lib.ref_random_descriptors(seed, n, nbytes, _p(out, _u8p))
        return out

    def default_pattern_text(self):
        n = self.lib.ref_default_pattern_text(None, 0)
        buf = C.create_string_buffer(n + 1)
        self.lib.ref_default_pattern_text(buf, n + 1)
        return buf.value.decode()

    def parse_pattern(self, text):
        T, K = C.c_int(), C.c_int()
        trip = np.zeros(6 * 8192, np.int32)
        weights = np.zeros(64 * 64, np.float64)
        self._check(self.lib.ref_parse_pattern(text.encode(), C.byref(T), C.byref(K),
                                               _p(trip, _i32p), trip.size, _p(weights, _f64p),
                                               weights.size))
        return (T.value, K.value, trip[:6 * T.value].reshape(-1, 6).copy(),
                weights[:K.value * K.value].copy())

    def load_pgm(self, path):
        w, h = C.c_int(), C.c_int()
        self._check(self.lib.ref_load_pgm(str(path).encode(), None, 0, C.byref(w), C.byref(h)))
        out = np.empty((h.value, w.value), np.float64)
        self._check(self.lib.ref_load_pgm(str(path).encode(), _p(out, _f64p), out.size,
                                          C.byref(w), C.byref(h)))
        return out

    def sample_candidates(self, count, K, seed):
        out = np.zeros((count, 6), np.int32)
        self._check(self.lib.ref_sample_candidates(count, K, seed, _p(out, _i32p)))
        return out

    def triplet_bits(self, windows, candidates, K, weights):
        windows = np.ascontiguousarray(windows, np.float64).reshape(-1, 4096)
        cand = np.ascontiguousarray(candidates, np.int32).reshape(-1, 6)
        weights = np.ascontiguousarray(weights, np.float64)
        n, c = len(windows), len(cand)
        row = (n + 7) // 8
        out = np.zeros((c, row), np.uint8)
        self._check(self.lib.ref_triplet_bits(_p(windows, _f64p), n, _p(cand, _i32p), c, K, _p(weights, _f64p),
                                              _p(out, _u8p), row))
        return out

    def detect(self, image, threshold=20.0, nms=True, orient=True):
        if orient:
            return self.detect_and_orient(image, threshold, nms)
        image = np.ascontiguousarray(image, np.float64)
        h, w = image.shape
        cap = max(w * h, 1)
        out = np.empty((cap, 4), np.float64)
        cnt = C.c_size_t()
        self._check(self.lib.ref_fast_detect(_p(image, _f64p), w, h, threshold, int(nms), _p(out, _f64p), cap,
                                             C.byref(cnt)))
        return out[:cnt.value].copy()

    def detect_and_orient(self, image, threshold=20.0, nms=True):
        image = np.ascontiguousarray(image, np.float64)
        h, w = image.shape
        cap = max(w * h, 1)
        out = np.empty((cap, 4), np.float64)
        cnt = C.c_size_t()
        self._check(self.lib.ref_detect_and_orient(_p(image, _f64p), w, h, threshold, int(nms),
                                                   _p(out, _f64p), cap, C.byref(cnt)))
        return out[:cnt.value].copy()

    def in_margin(self, w, h, x, y):
        return bool(self.lib.ref_keypoint_in_margin(w, h, x, y))

    def extract_window(self, image, kp):
        image = np.ascontiguousarray(image, np.float64)
        kp = np.ascontiguousarray(kp, np.float64)
        h, w = image.shape
        win = np.empty(4096, np.float64)
        self._check(self.lib.ref_extract_window(_p(image, _f64p), w, h, _p(kp, _f64p),
                                                _p(win, _f64p)))
        return win

    def oracle_window(self, image, kp):
        image = np.ascontiguousarray(image, np.float64)
        kp = np.ascontiguousarray(kp, np.float64)
        h, w = image.shape
        win = np.empty(4096, np.float64)
        self.lib.ref_oracle_window(_p(image, _f64p), w, h, _p(kp, _f64p), _p(win, _f64p))
        return win

    def triplet_bit(self, win, trip, K, weights):
        win = np.ascontiguousarray(win, np.float64)
        trip = np.ascontiguousarray(trip, np.int32)
        weights = np.ascontiguousarray(weights, np.float64)
        return bool(self.lib.ref_triplet_bit(_p(win, _f64p), _p(trip, _i32p), K,
                                             _p(weights, _f64p)))

    def describe(self, image, kp, pattern_text=None, scalar_oracle=False):
        image = np.ascontiguousarray(image, np.float64)
        kp = np.ascontiguousarray(kp, np.float64)
        h, w = image.shape
        out = np.zeros(1024, np.uint8)
        fn = self.lib.ref_oracle_describe if scalar_oracle else self.lib.ref_describe
        self._check(fn(_p(image, _f64p), w, h, _p(kp, _f64p),
                       pattern_text.encode() if pattern_text else None, _p(out, _u8p)))
        T = 512 if pattern_text is None else parse_pattern_text(pattern_text)[0]
        return out[:T // 8].copy()

    def describe_all(self, image, kps, pattern_text=None, workers=0):
        image = np.ascontiguousarray(image, np.float64)
        kps = np.ascontiguousarray(kps, np.float64)
        h, w = image.shape
        n = len(kps)
        T = 512 if pattern_text is None else parse_pattern_text(pattern_text)[0]
        kept = np.empty(n, np.int64)
        desc = np.zeros((n, T // 8), np.uint8)
        cnt = C.c_size_t()
        self._check(self.lib.ref_describe_all(_p(image, _f64p), w, h, _p(kps, _f64p), n,
                                              pattern_text.encode() if pattern_text else None,
                                              workers, _p(kept, _i64p), _p(desc, _u8p),
                                              C.byref(cnt)))
        return kept[:cnt.value].copy(), desc[:cnt.value].copy()

    def describe_all_file(self, image, kps):
        image = np.ascontiguousarray(image, np.float64)
        kps = np.ascontiguousarray(kps, np.float64)
        h, w = image.shape
        n = C.c_size_t()
        cap = 20 + len(kps) * 80
        buf = C.create_string_buffer(cap)
        self._check(self.lib.ref_describe_all_file(_p(image, _f64p), w, h, _p(kps, _f64p),
                                                   len(kps), buf, cap, C.byref(n)))
        return buf.raw[:n.value]

    def hamming(self, a, b):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.uint8)
        out = C.c_int()
        self._check(self.lib.ref_hamming(_p(a, _u8p), a.size, _p(b, _u8p), b.size, C.byref(out)))
        return out.value

    def knn2(self, probe, gallery):
        probe = np.ascontiguousarray(probe, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        out = np.empty(3, np.int32)
        nbytes = probe.size
        self._check(self.lib.ref_knn2(_p(probe, _u8p), _p(gallery, _u8p), len(gallery), nbytes,
                                      _p(out, _i32p)))
        return tuple(int(v) for v in out)

    def knn2_all(self, probes, gallery):
        probes = np.ascontiguousarray(probes, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        out = np.zeros((len(probes), 3), np.int32)
        self._check(self.lib.ref_knn2_all(_p(probes, _u8p), len(probes), _p(gallery, _u8p),
                                          len(gallery), probes.shape[1], _p(out, _i32p)))
        return out

    def match(self, probes, gallery, ratio=None, cross_check=False, max_distance=None,
              workers=0, scalar_oracle=False):
        probes = np.ascontiguousarray(probes, np.uint8)
        gallery = np.ascontiguousarray(gallery, np.uint8)
        q, n = len(probes), len(gallery)
        nbytes = probes.shape[1]
        out = np.empty((max(q, 1), 4), np.int32)
        cnt = C.c_size_t()
        if scalar_oracle:
            rc = self.lib.ref_oracle_match(_p(probes, _u8p), q, _p(gallery, _u8p), n, nbytes,
                                           int(ratio is not None), float(ratio or 0.0),
                                           int(cross_check), int(max_distance is not None),
                                           int(max_distance or 0), _p(out, _i32p), C.byref(cnt))
        else:
            rc = self.lib.ref_match(_p(probes, _u8p), q, _p(gallery, _u8p), n, nbytes,
                                    int(ratio is not None), float(ratio or 0.0), int(cross_check),
                                    int(max_distance is not None), int(max_distance or 0),
                                    workers, _p(out, _i32p), C.byref(cnt))
        self._check(rc)
        return out[:cnt.value].copy()


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref():
    """The unmodified reference, or None if oracle/_ref has not been built."""
    global _ref
    if _ref is None and REF_SO.exists():
        _ref = Ref()
    return _ref


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
