"""B200-native CLATCH: LATCH descriptor extraction and Hamming top-2 matching.

Drop-in for the two hot paths of the reference package ``latchkit``
(proj/python/latchkit/__init__.py:10-25, proj/bindings/module.cpp:204-248):
``describe``, ``match`` and ``hamming`` keep the reference's signatures, array
shapes/dtypes and exception types, and produce bit-identical results; the work
runs in hand-written sm_100a kernels behind the C ABI in include/clatch.h.

``detect`` (FAST-9 + NMS + orientation, the step before the path) and the LTCH descriptor
container (the file between the reference's ``latch describe`` and ``latch match``) are provided as well.
Not provided (outside the hot path): evaluate, train, warp, load_pgm, save_pgm — keep using the reference's host code for those.
"""
from __future__ import annotations

import numpy as np

from ._lib import ClatchDeviceError, LatchError
from .container import format_descriptor_file, load_descriptor_file, parse_descriptor_file, save_descriptor_file
from .engine import DescriptorSet, Engine, get_engine
from .pattern import (TripletPattern, default_pattern as _default_pattern, default_pattern_text,
                      format_pattern, parse_pattern, pattern_from_text)

# Module constants, bindings/module.cpp:208-211.
descriptor_bits = 512
descriptor_bytes = 64
window_margin = 46
orientation_radius = 15

__all__ = [
    "default_pattern", "describe", "describe_batch", "descriptor_bits", "detect", "descriptor_bytes", "hamming", "match",
    "orientation_radius", "window_margin", "Engine", "DescriptorSet", "get_engine", "LatchError",
    "ClatchDeviceError", "TripletPattern", "parse_pattern", "format_pattern",
    "format_descriptor_file", "parse_descriptor_file", "save_descriptor_file", "load_descriptor_file",
]


def default_pattern() -> str:
    """Text of the built-in 512-triplet pattern (bindings/module.cpp:245-247)."""
    return default_pattern_text()


def _image_array(image) -> np.ndarray:
    # image_from_array, bindings/module.cpp:33-41 (+ uint8 accepted as-is: lossless and 8x
    # less to upload; every PGM-sourced image is integer valued, src/image.cpp:75-76).
    a = np.asarray(image)
    if a.ndim != 2:
        raise ValueError("image must be a 2d array")
    if a.shape[0] <= 0 or a.shape[1] <= 0:
        raise ValueError("image must be non-empty")
    if a.dtype != np.uint8:
        a = np.ascontiguousarray(a, dtype=np.float64)   # c_style | forcecast
    return a


def _keypoint_array(keypoints) -> np.ndarray:
    # keypoints_from_array, bindings/module.cpp:49-62
    a = np.ascontiguousarray(keypoints, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] < 2 or a.shape[1] > 4:
        raise ValueError("keypoints must be (N, 2..4): x, y[, theta[, score]]")
    return a


def _descriptor_array(a, what: str) -> np.ndarray:
    # descriptors_from_array, bindings/module.cpp:76-86 (ByteArray: uint8, no forcecast)
    a = np.asarray(a)
    if a.dtype != np.uint8:
        raise TypeError(f"{what} must be a uint8 array")
    if a.ndim != 2:
        raise ValueError(f"{what} must be a (N, descriptor_bytes) uint8 array")
    return np.ascontiguousarray(a)


def detect(image, threshold=20.0, nms=True, orient=True):
    """FAST-9 corners as an (N, 4) array [x, y, theta, score] — latchkit.detect
    (bindings/module.cpp:100-105 -> fast_detect / detect_and_orient, src/detect.cpp:76-157).
    With orient, theta is the intensity-centroid angle (radius 15) and detections whose
    orientation disc leaves the image are dropped. Images smaller than 7x7 raise RuntimeError."""
    return get_engine().detect(_image_array(image), threshold, nms, orient, orientation_radius)


def describe(image, keypoints, pattern=None, workers=0):
    """Binary descriptors for the keypoints that keep the 46 px window margin.

    Same contract as latchkit.describe (bindings/module.cpp:106-121 -> describe_all,
    src/descriptor.cpp:90-105): returns ``(kept_keypoints (M,4) float64, descriptors
    (M, T/8) uint8)``; margin violators are dropped silently, input order is kept;
    ``pattern`` is pattern-file text or None for the built-in arrangement; missing
    theta/score columns read as 0. ``workers`` only sizes the host-side trig pass —
    results never depend on it.
    """
    img = _image_array(image)
    pat = pattern_from_text(pattern)
    kps = _keypoint_array(keypoints)
    eng = get_engine()
    kept, desc = eng.describe_all(img, kps, workers, pattern=pat)     # pattern installed under the launch's lock
    return eng.take_keypoints(kps, kept, workers), desc


def describe_batch(images, keypoints, pattern=None, workers=0):
    """describe() over a list of images and keypoint arrays in one pipelined call (extension
    for the many-images-per-GPU workload). Returns a list of (kept_keypoints, descriptors),
    each identical to describe(images[i], keypoints[i], pattern)."""
    pat = pattern_from_text(pattern)
    imgs = [_image_array(im) for im in images]
    kps = [_keypoint_array(k) for k in keypoints]
    if len(imgs) != len(kps):
        raise ValueError("describe_batch needs one keypoint array per image")
    if len({im.dtype for im in imgs}) > 1:          # mixed input: use the reference dtype for all
        imgs = [np.ascontiguousarray(im, dtype=np.float64) for im in imgs]
    widest = max((k.shape[1] for k in kps), default=4)
    if any(k.shape[1] != widest for k in kps):
        kps = [np.hstack([k, np.zeros((len(k), widest - k.shape[1]))]) for k in kps]
    eng = get_engine()
    res = eng.describe_batch(imgs, kps, workers, pattern=pat)
    return [(eng.take_keypoints(k, kept, workers), desc) for k, (kept, desc) in zip(kps, res)]


def match(probes, gallery, ratio=None, cross_check=False, max_distance=None, workers=0):
    """Brute-force Hamming matches as an (M, 4) int32 array
    [probe, gallery, distance, second_distance] — latchkit.match
    (bindings/module.cpp:123-144 -> match_brute_force, src/match.cpp:52-81).
    Empty gallery raises RuntimeError (EmptyGallery) even with no probes; empty
    probes give a (0, 4) array. ``workers`` is accepted for compatibility."""
    p = _descriptor_array(probes, "probes")
    g = _descriptor_array(gallery, "gallery")
    if len(g) == 0:
        raise LatchError("EmptyGallery", "matching needs a nonempty gallery")
    if len(p) == 0:
        return np.zeros((0, 4), np.int32)
    if p.shape[1] != g.shape[1]:
        raise LatchError("LengthMismatch",
                         f"descriptor lengths differ: {p.shape[1]} vs {g.shape[1]}")
    return get_engine().match_brute_force(p, g, ratio=ratio, cross_check=cross_check,
                                          max_distance=max_distance)


def hamming(a, b) -> int:
    """Hamming distance between two equal-length uint8 rows (bindings/module.cpp:146-153 ->
    src/match.cpp:14-31). Runs the device matcher on a 1x1 problem — the product has
    no CPU arithmetic path, so this is a correctness entry point, not a fast one."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim != 1 or b.ndim != 1:
        raise ValueError("hamming expects two 1d uint8 arrays")
    if a.dtype != np.uint8 or b.dtype != np.uint8:
        raise TypeError("hamming expects uint8 arrays")
    if a.shape[0] != b.shape[0]:
        raise LatchError("LengthMismatch",
                         f"descriptor lengths differ: {a.shape[0]} vs {b.shape[0]}")
    if a.shape[0] == 0:
        return 0
    _, dist, _ = get_engine().match_top2(a.reshape(1, -1), b.reshape(1, -1))
    return int(dist[0])
