"""LTCH descriptor container (the reference's `latch describe` output / `latch match` input):
read and write it straight from the arrays describe() returns, so a file-based pipeline can
switch to the GPU path without touching its files.

Layout (proj/src/descriptor.cpp:110-194, little-endian): magic "LTCH", u32 version = 1,
u32 record count, u32 descriptor bytes, u32 reserved = 0, then per record four float32
(x, y, theta, score — the float64 keypoint fields narrowed exactly as `static_cast<float>`
does) followed by the descriptor bytes. Errors mirror the reference's categories (BadHeader,
Truncated, Malformed) as RuntimeError, the way pybind11 surfaces latch::Error.
"""
from __future__ import annotations

import numpy as np

from ._lib import LatchError

MAGIC = b"LTCH"
VERSION = 1
_HEADER = np.dtype([("version", "<u4"), ("count", "<u4"), ("bytes", "<u4"), ("reserved", "<u4")])


def format_descriptor_file(keypoints, descriptors) -> bytes:
    """format_descriptor_file (descriptor.cpp:146-162). keypoints: (M, 4) float array
    [x, y, theta, score]; descriptors: (M, B) uint8. An empty set writes B = 0, like the reference."""
    kps = np.asarray(keypoints, dtype=np.float64)
    desc = np.asarray(descriptors)
    if desc.dtype != np.uint8:
        raise TypeError("descriptors must be a uint8 array")
    if kps.ndim != 2 or kps.shape[1] != 4 or desc.ndim != 2 or len(kps) != len(desc):
        raise ValueError("expected keypoints (M, 4) and descriptors (M, B) with the same M")
    count = len(desc)
    nbytes = desc.shape[1] if count else 0
    head = np.zeros(1, _HEADER)
    head["version"], head["count"], head["bytes"] = VERSION, count, nbytes
    records = np.empty((count, 16 + nbytes), np.uint8)
    with np.errstate(over="ignore"):                       # a double beyond float range narrows to inf, as in C++
        records[:, :16] = kps.astype("<f4").view(np.uint8).reshape(count, 16)
    if count:
        records[:, 16:] = desc
    return MAGIC + head.tobytes() + records.tobytes()


def parse_descriptor_file(blob: bytes):
    """parse_descriptor_file (descriptor.cpp:164-194) -> (keypoints (M, 4) float64, descriptors (M, B) uint8)."""
    blob = bytes(blob)
    if len(blob) < 4 or blob[:4] != MAGIC:
        raise LatchError("BadHeader", "not a descriptor file (bad magic)")
    if len(blob) < 4 + _HEADER.itemsize:
        raise LatchError("Truncated", "descriptor file ends mid-field")
    head = np.frombuffer(blob, _HEADER, 1, 4)[0]
    if int(head["version"]) != VERSION:
        raise LatchError("BadHeader", f"unsupported descriptor file version {int(head['version'])}")
    count, nbytes = int(head["count"]), int(head["bytes"])
    body = len(blob) - 4 - _HEADER.itemsize
    record = 16 + nbytes
    if body < count * record:
        # the reference reads record by record: a cut inside the four floats is "mid-field",
        # one inside the descriptor bytes is "mid-record"
        mid_field = (body % record) < 16 if record else True
        raise LatchError("Truncated", "descriptor file ends mid-field" if mid_field else
                         "descriptor file ends mid-record")
    rec = np.frombuffer(blob, np.uint8, count * record, 4 + _HEADER.itemsize).reshape(count, record)
    kps = rec[:, :16].copy().view("<f4").reshape(count, 4).astype(np.float64)
    return kps, rec[:, 16:].copy()


def save_descriptor_file(keypoints, descriptors, path) -> None:
    """save_descriptor_file (descriptor.cpp:196-202)."""
    data = format_descriptor_file(keypoints, descriptors)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise LatchError("Malformed", f"cannot open '{path}' for writing") from e


def load_descriptor_file(path):
    """load_descriptor_file (descriptor.cpp:204-211)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise LatchError("Malformed", f"cannot open '{path}'") from e
    return parse_descriptor_file(data)
