"""One CLATCH context per GPU: the Python face of include/clatch.h.

`Engine` owns a clatch_ctx (device, stream, scratch) and exposes both forms of the
ABI: host-buffer calls on numpy arrays (what the reference-facing API uses) and
device-resident calls on torch CUDA tensors (torch is only the allocator / stream
provider here — the kernels are libclatch.so's own).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

from . import _lib
from ._lib import f64p, i16p, i32p, i64p, u8p
from .pattern import TripletPattern, default_pattern


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class _PinnedPool:
    """Result arrays for describe() / describe_batch(). Page-locked memory makes both of their trips
    over the bus plain DMAs (descriptor arrays usually come straight back as match() inputs, and a
    batch call's downloads never stall its pipeline) — but cudaHostAlloc costs about 3 ms per MB on
    the B200 hosts, ten times what first-touching pageable memory costs. So page-locked blocks are
    handed out only where they will be recycled:

    * blocks are kept by power-of-two size and reused; a block returns to the pool when the last
      numpy view of it dies;
    * a NEW block is allocated only after an earlier result of that size has been released (a loop
      that drops its previous result: the second iteration pays the allocation, the rest reuse it);
    * a caller that keeps every result gets ordinary pageable arrays, and so does anyone beyond
      `max_live_bytes` of outstanding page-locked memory.
    """

    def __init__(self, lib, max_live_bytes: int = 1 << 30):
        self.lib, self.free, self.released, self.live_bytes = lib, {}, {}, 0
        self.max_live_bytes = max_live_bytes
        self.lock = threading.Lock()

    def empty(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        count = int(np.prod(shape))
        cap = 1 << max(12, (max(count * dtype.itemsize, 1) - 1).bit_length())
        with self.lock:
            blocks = self.free.get(cap)
            ptr = blocks.pop() if blocks else None
            if ptr is None:
                if self.released.get(cap, 0) <= 0 or self.live_bytes + cap > self.max_live_bytes:
                    ptr = False                       # no evidence of recycling (or over budget): pageable
                else:
                    self.released[cap] -= 1
            if ptr is not False:
                self.live_bytes += cap
        if ptr is False:
            arr = np.empty(shape, dtype)
            weakref.finalize(arr, self._note_release, cap)
            return arr
        if ptr is None:
            p = C.c_void_p()
            rc = self.lib.clatch_host_alloc(cap, C.byref(p))
            if rc != 0 or not p.value:
                with self.lock:
                    self.live_bytes -= cap
                return np.empty(shape, dtype)
            ptr = p.value
        owner = (C.c_uint8 * cap).from_address(ptr)
        weakref.finalize(owner, self._release, ptr, cap)
        return np.frombuffer(owner, dtype=dtype, count=count).reshape(shape)

    def _note_release(self, cap):
        with self.lock:
            self.released[cap] = self.released.get(cap, 0) + 1

    def _release(self, ptr, cap):
        with self.lock:
            self.live_bytes -= cap
            self.free.setdefault(cap, []).append(ptr)


class DescriptorSet:
    """Device-resident set of 64-byte descriptors (clatch_set): uploaded / copied once, kept with
    its tensor-core operand forms, reusable across any number of matches."""

    def __init__(self, engine: "Engine", handle, count: int):
        self.engine, self.handle, self.count = engine, handle, count

    def __len__(self):
        return self.count

    def close(self):
        if self.handle:
            self.engine.lib.clatch_set_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    def __init__(self, device: int | None = None):
        self.lib = _lib.load()
        if device is None:
            device = int(os.environ.get("CLATCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        handle = C.c_void_p()
        _lib.check(self.lib.clatch_ctx_create(int(device), C.byref(handle)))
        self.ctx = handle
        self.device = int(device)
        self._pattern_key = None
        self._pattern = None
        self._lock = threading.RLock()      # serialises every ABI call on this context (and its pattern)
        self._pinned = _PinnedPool(self.lib)
        sm, khz = C.c_int(), C.c_int()
        name = C.create_string_buffer(256)
        _lib.check(self.lib.clatch_device_info(self.ctx, C.byref(sm), C.byref(khz), name, 256))
        self.sm_count, self.sm_clock_khz, self.name = sm.value, khz.value, name.value.decode()

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.clatch_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- pattern ---------------------------------------------------------
    def set_pattern(self, pattern: TripletPattern | None = None) -> TripletPattern:
        """Install `pattern` (None = the built-in table) on the context. The pattern is context state:
        callers that must extract with a particular pattern pass it to describe_all / describe_batch /
        extract, which install it and launch under one hold of the context lock."""
        pattern = pattern or default_pattern()
        with self._lock:
            if pattern is self._pattern:
                return pattern
            key = pattern.key()
            if key != self._pattern_key:
                trip = np.ascontiguousarray(pattern.triplets, np.int16)
                w = np.ascontiguousarray(pattern.weights, np.float64)
                _lib.check(self.lib.clatch_set_pattern(self.ctx, _ptr(trip, i16p), pattern.bit_count,
                                                       pattern.patch_size, _ptr(w, f64p)))
                self._pattern_key = key
            self._pattern = pattern
        return pattern

    @property
    def descriptor_bytes(self) -> int:
        return int(self.lib.clatch_descriptor_bytes(self.ctx))

    @property
    def launch_count(self) -> int:
        return int(self.lib.clatch_launch_count(self.ctx))

    def set_option(self, key: str, value: int):
        """Tuning knobs that never change results, e.g. set_option("match_variant", 3)."""
        _lib.check(self.lib.clatch_set_option(self.ctx, key.encode(), int(value)))

    def synchronize(self):
        _lib.check(self.lib.clatch_synchronize(self.ctx))

    def extract_stats(self) -> tuple[int, int]:
        """(triplets recomputed exactly, warp passes through the exact path) of the filtered
        extraction kernel since set_option("extract_stats", 1)."""
        a, b = C.c_uint64(), C.c_uint64()
        _lib.check(self.lib.clatch_extract_stats(self.ctx, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    # ---- host-side preparation ----------------------------------------------
    def prepare_keypoints(self, keypoints: np.ndarray, width: int, height: int, workers: int = 0):
        """-> (xycs float64 (M,4) = x, y, cos, sin; kept int64 (M,) input indices)."""
        kps = np.ascontiguousarray(keypoints, np.float64)
        n, cols = kps.shape
        xycs = np.empty((n, 4), np.float64)
        kept = np.empty(n, np.int64)
        m = C.c_size_t()
        _lib.check(self.lib.clatch_prepare_keypoints(_ptr(kps, f64p), n, cols, width, height, workers,
                                                     _ptr(xycs, f64p), _ptr(kept, i64p), C.byref(m)))
        return xycs[:m.value], kept[:m.value]

    def take_keypoints(self, keypoints: np.ndarray, kept: np.ndarray, workers: int = 0) -> np.ndarray:
        """(M, 4) float64 rows keypoints[kept] with missing theta / score columns read as 0."""
        kps = np.ascontiguousarray(keypoints, np.float64)
        idx = np.ascontiguousarray(kept, np.int64)
        out = np.empty((len(idx), 4), np.float64)
        _lib.check(self.lib.clatch_take_keypoints(_ptr(kps, f64p), kps.shape[1], _ptr(idx, i64p), len(idx), workers,
                                                  _ptr(out, f64p)))
        return out

    # ---- detection ----------------------------------------------------------------------
    def detect(self, image: np.ndarray, threshold: float = 20.0, nms: bool = True, orient: bool = True,
               radius: int = 15) -> np.ndarray:
        """FAST-9 (+ NMS, + intensity-centroid angle) -> (N, 4) float64 [x, y, theta, score]."""
        h, w = image.shape
        image, pitch = self._rows(image)
        if image.dtype == np.uint8:
            fn, ptr = self.lib.clatch_detect_u8, _ptr(image, u8p)
        elif image.dtype == np.float64:
            fn, ptr = self.lib.clatch_detect_f64, _ptr(image, f64p)
        else:
            raise TypeError("image dtype must be uint8 or float64")
        cap = max(1024, (w * h) // 64)
        count = C.c_size_t()
        while True:
            out = np.empty((cap, 4), np.float64)
            with self._lock:
                rc = fn(self.ctx, ptr, w, h, pitch, float(threshold), int(nms), int(orient), int(radius),
                        _ptr(out, f64p), cap, C.byref(count))
            if rc == _lib.ERR_INVALID and count.value > cap:
                cap = count.value
                continue
            _lib.check(rc)
            return out[:count.value].copy()

    # ---- extraction, host buffers --------------------------------------------
    @staticmethod
    def _rows(image: np.ndarray):
        """(image with unit inner stride and a positive whole-element row pitch, pitch in elements).
        Anything else — transposed, negative or overlapping strides (img[::-1], broadcast views) — is copied."""
        h, w = image.shape
        if (image.strides[1] != image.itemsize or image.strides[0] % image.itemsize
                or image.strides[0] < w * image.itemsize):
            image = np.ascontiguousarray(image)
        return image, image.strides[0] // image.itemsize

    def extract(self, image: np.ndarray, xycs: np.ndarray, out: np.ndarray | None = None,
                pattern: TripletPattern | None = None) -> np.ndarray:
        """image: 2-D uint8 or float64 (rows may be strided); xycs from prepare_keypoints."""
        m = len(xycs)
        h, w = image.shape
        image, pitch = self._rows(image)
        xycs = np.ascontiguousarray(xycs, np.float64)
        with self._lock:
            if pattern is not None:
                self.set_pattern(pattern)
            if out is None:
                out = np.empty((m, self.descriptor_bytes), np.uint8)
            if image.dtype == np.uint8:
                rc = self.lib.clatch_extract_u8(self.ctx, _ptr(image, u8p), w, h, pitch,
                                                _ptr(xycs, f64p), m, _ptr(out, u8p))
            elif image.dtype == np.float64:
                rc = self.lib.clatch_extract_f64(self.ctx, _ptr(image, f64p), w, h, pitch,
                                                 _ptr(xycs, f64p), m, _ptr(out, u8p))
            else:
                raise TypeError("image dtype must be uint8 or float64")
        _lib.check(rc)
        return out

    def describe_all(self, image: np.ndarray, keypoints: np.ndarray, workers: int = 0,
                     pattern: TripletPattern | None = None):
        """describe_all in one ABI call: -> (kept int64 (M,), descriptors uint8 (M, T/8)). `pattern`
        (when given) is installed under the same hold of the context lock as the launch, so concurrent
        callers with different patterns cannot swap it in between."""
        h, w = image.shape
        image, pitch = self._rows(image)
        kps = np.ascontiguousarray(keypoints, np.float64)
        n, cols = kps.shape
        kept = np.empty(n, np.int64)
        m = C.c_size_t()
        with self._lock:
            if pattern is not None:
                self.set_pattern(pattern)
            out = self._pinned.empty((n, self.descriptor_bytes), np.uint8)
            if image.dtype == np.uint8:
                rc = self.lib.clatch_describe_all_u8(self.ctx, _ptr(image, u8p), w, h, pitch, _ptr(kps, f64p),
                                                     n, cols, workers, _ptr(kept, i64p), _ptr(out, u8p),
                                                     C.byref(m))
            elif image.dtype == np.float64:
                rc = self.lib.clatch_describe_all_f64(self.ctx, _ptr(image, f64p), w, h, pitch,
                                                      _ptr(kps, f64p), n, cols, workers, _ptr(kept, i64p),
                                                      _ptr(out, u8p), C.byref(m))
            else:
                raise TypeError("image dtype must be uint8 or float64")
        _lib.check(rc)
        return kept[:m.value], out[:m.value]

    def describe_batch(self, images, keypoints, workers: int = 0, pattern: TripletPattern | None = None):
        """describe_all over many images in one pipelined ABI call. images: list of 2-D arrays, all
        uint8 or all float64; keypoints: list of (N_i, cols) float64 arrays with one common cols.
        -> list of (kept int64 (M_i,), descriptors uint8 (M_i, T/8))."""
        n_img = len(images)
        if n_img == 0:
            return []
        dtype = images[0].dtype
        imgs, kps_l = [], []
        for im in images:
            if im.dtype != dtype:
                raise TypeError("describe_batch needs one image dtype per call")
            imgs.append(self._rows(im)[0])
        for k in keypoints:
            kps_l.append(np.ascontiguousarray(k, np.float64))
        cols = kps_l[0].shape[1]
        if any(k.shape[1] != cols for k in kps_l):
            raise ValueError("describe_batch needs one keypoint column count per call")
        kept = [np.empty(len(k), np.int64) for k in kps_l]
        vp = C.c_void_p * n_img
        widths = (C.c_int * n_img)(*[im.shape[1] for im in imgs])
        heights = (C.c_int * n_img)(*[im.shape[0] for im in imgs])
        pitches = (C.c_size_t * n_img)(*[im.strides[0] // im.itemsize for im in imgs])
        counts = (C.c_size_t * n_img)(*[len(k) for k in kps_l])
        m = (C.c_size_t * n_img)()
        fn = {np.dtype(np.uint8): self.lib.clatch_describe_batch_u8,
              np.dtype(np.float64): self.lib.clatch_describe_batch_f64}.get(np.dtype(dtype))
        if fn is None:
            raise TypeError("image dtype must be uint8 or float64")
        with self._lock:
            if pattern is not None:
                self.set_pattern(pattern)
            nbytes = self.descriptor_bytes
            out = [self._pinned.empty((len(k), nbytes), np.uint8) for k in kps_l]   # page-locked: direct DMA targets
            rc = fn(self.ctx, vp(*[im.ctypes.data for im in imgs]), widths, heights, pitches,
                    vp(*[k.ctypes.data for k in kps_l]), counts, cols, n_img, workers,
                    vp(*[a.ctypes.data for a in kept]), vp(*[a.ctypes.data for a in out]), m)
        _lib.check(rc)
        return [(kept[i][:m[i]], out[i][:m[i]]) for i in range(n_img)]

    # ---- extraction, device tensors --------------------------------------------
    def extract_device(self, image, xycs, out=None, stream=None):
        """image: torch CUDA tensor (H, W) uint8 or float64, unit inner stride; xycs: CUDA
        float64 (M, 4). Queues on `stream` (default: torch's current stream); no sync."""
        import torch
        assert image.is_cuda and xycs.is_cuda and image.dim() == 2 and image.stride(1) == 1
        m = xycs.shape[0]
        if out is None:
            out = torch.empty((m, self.descriptor_bytes), dtype=torch.uint8, device=image.device)
        st = (stream or torch.cuda.current_stream(image.device)).cuda_stream
        h, w = image.shape
        fn = {torch.uint8: self.lib.clatch_extract_u8_dev,
              torch.float64: self.lib.clatch_extract_f64_dev}[image.dtype]
        _lib.check(fn(self.ctx, image.data_ptr(), w, h, image.stride(0), xycs.data_ptr(), m,
                      out.data_ptr(), st))
        return out

    def estimate_planes_device(self, image, xycs, stream=None):
        """Diagnostics: the 64 x 64 samples (uint16, round(256 * v)) the default extraction kernel's estimate works
        from, for a uint8 CUDA image and prepared keypoint records — (M, 64, 64) on the device."""
        import torch
        assert image.is_cuda and xycs.is_cuda and image.dtype == torch.uint8 and image.stride(1) == 1
        m = xycs.shape[0]
        out = torch.empty((m, 64, 64), dtype=torch.int16, device=image.device)
        st = (stream or torch.cuda.current_stream(image.device)).cuda_stream
        h, w = image.shape
        with self._lock:
            _lib.check(self.lib.clatch_estimate_planes_u8_dev(self.ctx, image.data_ptr(), w, h, image.stride(0),
                                                              xycs.data_ptr(), m, out.data_ptr(), st))
        return out

    # ---- matching, host buffers ------------------------------------------------
    def match_top2(self, queries: np.ndarray, train: np.ndarray):
        """-> (best_idx, best_dist, second_dist) int32 (Q,) each."""
        q = np.ascontiguousarray(queries, np.uint8)
        t = q if train is queries else np.ascontiguousarray(train, np.uint8)
        nq, nt = len(q), len(t)
        nbytes = q.shape[1] if q.ndim == 2 else t.shape[1]
        res = np.empty((3, nq), np.int32)
        with self._lock:
            rc = self.lib.clatch_match_top2(self.ctx, _ptr(q, u8p), nq, _ptr(t, u8p), nt, nbytes,
                                            _ptr(res[0], i32p), _ptr(res[1], i32p), _ptr(res[2], i32p))
        _lib.check(rc)
        return res[0], res[1], res[2]

    def match_brute_force(self, probes: np.ndarray, gallery: np.ndarray, ratio=None,
                          cross_check=False, max_distance=None) -> np.ndarray:
        """-> int32 (M, 4) rows [probe, gallery, distance, second_distance]."""
        p = np.ascontiguousarray(probes, np.uint8)
        g = np.ascontiguousarray(gallery, np.uint8)
        nq, nt = len(p), len(g)
        out = np.empty((max(nq, 1), 4), np.int32)
        count = C.c_size_t()
        with self._lock:
            rc = self.lib.clatch_match_brute_force(
                self.ctx, _ptr(p, u8p), nq, _ptr(g, u8p), nt, p.shape[1],
                int(ratio is not None), float(ratio) if ratio is not None else 0.0, int(cross_check),
                int(max_distance is not None), int(max_distance) if max_distance is not None else 0,
                _ptr(out, i32p), C.byref(count))
        _lib.check(rc)
        return out[:count.value].copy()

    def filter_matches(self, best_idx, best_dist, second_dist, ratio=None, max_distance=None,
                       reverse_best=None) -> np.ndarray:
        bi = np.ascontiguousarray(best_idx, np.int32)
        bd = np.ascontiguousarray(best_dist, np.int32)
        sd = np.ascontiguousarray(second_dist, np.int32)
        rb = None if reverse_best is None else np.ascontiguousarray(reverse_best, np.int32)
        nq = len(bi)
        out = np.empty((max(nq, 1), 4), np.int32)
        count = C.c_size_t()
        _lib.check(self.lib.clatch_filter_matches(
            _ptr(bi, i32p), _ptr(bd, i32p), _ptr(sd, i32p), nq, int(ratio is not None),
            float(ratio) if ratio is not None else 0.0, int(max_distance is not None),
            int(max_distance) if max_distance is not None else 0,
            None if rb is None else _ptr(rb, i32p), _ptr(out, i32p), C.byref(count)))
        return out[:count.value].copy()

    # ---- trainer scoring ----------------------------------------------------------------
    def triplet_bits(self, windows: np.ndarray, candidates: np.ndarray, patch_size: int = 8, mask=None):
        """bit (c, i) = triplet_bit(window i, candidate c, mask): windows (n, 64, 64) float64 upright
        patches, candidates (C, 6) ints -> uint8 (C, ceil(n/8)), LSB-first (BitVector order)."""
        w = np.ascontiguousarray(windows, np.float64).reshape(-1, 4096)
        cand = np.ascontiguousarray(candidates, np.int16).reshape(-1, 6)
        m = None if mask is None else np.ascontiguousarray(mask, np.float64).reshape(-1)
        if m is not None and m.size != patch_size * patch_size:
            raise ValueError("mask must hold patch_size * patch_size weights")
        n, c = len(w), len(cand)
        row = (n + 7) // 8
        out = np.zeros((c, row), np.uint8)
        with self._lock:
            rc = self.lib.clatch_triplet_bits(self.ctx, _ptr(w, f64p), n, _ptr(cand, i16p), c, int(patch_size),
                                              None if m is None else _ptr(m, f64p), _ptr(out, u8p), row)
        _lib.check(rc)
        return out

    # ---- resident descriptor sets ----------------------------------------------------
    def create_set(self, descriptors) -> DescriptorSet:
        """descriptors: (N, 64) uint8 numpy array (uploaded) or torch CUDA tensor (copied on device)."""
        handle = C.c_void_p()
        if isinstance(descriptors, np.ndarray):
            d = np.ascontiguousarray(descriptors, np.uint8)
            if d.ndim != 2 or d.shape[1] != 64:
                raise ValueError("descriptor sets hold (N, 64) uint8 rows")
            with self._lock:
                rc = self.lib.clatch_set_create(self.ctx, d.ctypes.data, len(d), 0, C.byref(handle))
            n = len(d)
        else:
            import torch
            d = descriptors.contiguous()
            if d.dim() != 2 or d.shape[1] != 64 or d.dtype != torch.uint8 or not d.is_cuda:
                raise ValueError("descriptor sets hold (N, 64) uint8 rows")
            torch.cuda.current_stream(d.device).synchronize()   # the copy runs on the context's stream
            with self._lock:
                rc = self.lib.clatch_set_create(self.ctx, d.data_ptr(), d.shape[0], 1, C.byref(handle))
            n = d.shape[0]
        _lib.check(rc)
        return DescriptorSet(self, handle, n)

    def match_sets(self, probes: DescriptorSet, gallery: DescriptorSet, ratio=None, cross_check=False,
                   max_distance=None) -> np.ndarray:
        out = np.empty((max(len(probes), 1), 4), np.int32)
        count = C.c_size_t()
        with self._lock:
            rc = self.lib.clatch_match_sets(
                self.ctx, probes.handle, gallery.handle, int(ratio is not None),
                float(ratio) if ratio is not None else 0.0, int(cross_check), int(max_distance is not None),
                int(max_distance) if max_distance is not None else 0, _ptr(out, i32p), C.byref(count))
        _lib.check(rc)
        return out[:count.value].copy()

    def match_set_pairs(self, sets, pairs, ratio=None, cross_check=False, max_distance=None):
        """All (probe set, gallery set) index pairs in as few launches as memory allows.
        -> list of (M_p, 4) int32 arrays, one per pair, in the order given."""
        pairs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
        handles = (C.c_void_p * len(sets))(*[s.handle for s in sets])
        cap = int(sum(len(sets[i]) for i in pairs[:, 0])) if len(pairs) else 0
        out = np.empty((max(cap, 1), 4), np.int32)
        offsets = np.zeros(len(pairs) + 1, np.uintp)
        with self._lock:
            rc = self.lib.clatch_match_set_pairs(
                self.ctx, handles, len(sets), _ptr(pairs, i32p), len(pairs), int(ratio is not None),
                float(ratio) if ratio is not None else 0.0, int(cross_check), int(max_distance is not None),
                int(max_distance) if max_distance is not None else 0, _ptr(out, i32p), cap,
                offsets.ctypes.data_as(_lib.szp))
        _lib.check(rc)
        return [out[int(offsets[p]):int(offsets[p + 1])] for p in range(len(pairs))]

    # ---- matching, device tensors ------------------------------------------------
    def match_top2_device(self, queries, train, out=None, stream=None):
        """queries (Q, B), train (N, B): contiguous CUDA uint8 tensors. Returns an int32 CUDA
        tensor (3, Q): rows best_idx, best_dist, second_dist. Queued, not synchronised."""
        import torch
        assert queries.is_cuda and train.is_cuda and queries.is_contiguous() and train.is_contiguous()
        nq, nbytes = queries.shape
        if out is None:
            out = torch.empty((3, nq), dtype=torch.int32, device=queries.device)
        st = (stream or torch.cuda.current_stream(queries.device)).cuda_stream
        _lib.check(self.lib.clatch_match_top2_dev(
            self.ctx, queries.data_ptr(), nq, train.data_ptr(), train.shape[0], nbytes,
            out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), st))
        return out


_engines: dict[int, Engine] = {}
_engines_lock = threading.Lock()


def get_engine(device: int | None = None) -> Engine:
    """Process-wide engine for `device` (default CLATCH_DEVICE / LOCAL_RANK / 0)."""
    if device is None:
        device = int(os.environ.get("CLATCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _engines_lock:
        eng = _engines.get(device)
        if eng is None:
            eng = _engines[device] = Engine(device)
        return eng
