"""Host-side pattern handling: the LATCHPAT v1 text format and the built-in table.

Mirrors the reference's parse_pattern / format_pattern / default_pattern
(proj/src/pattern.cpp:68-155, proj/src/pattern_default.cpp:527-539): same accepted
syntax, same error categories (surfaced as RuntimeError, as pybind11 does for
latch::Error). The shipped table lives in data/default_pattern.npz (int16 triplets + f64
weights, taken from the reference's own format_pattern(default_pattern()) output by
oracle/make_golden.py); its LATCHPAT text is produced on demand by format_pattern.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

import numpy as np

from ._lib import LatchError

WINDOW = 64          # proj/include/latch/pattern.hpp:12
_DATA = Path(__file__).resolve().parent / "data" / "default_pattern.npz"
_TEXT_CACHE = Path(__file__).resolve().parent / "data" / "default_pattern.latchpat"   # generated, git-ignored
_HEADER = re.compile(r"LATCHPAT v1 T=\s*([+-]?\d+) K=\s*([+-]?\d+)")
_INT = re.compile(r"\s*([+-]?\d+)")


@dataclass(frozen=True)
class TripletPattern:
    """T triplets {ax, ay, bx, by, cx, cy} + K*K weights (pattern.hpp:19-52)."""
    bit_count: int
    patch_size: int
    triplets: np.ndarray   # int16 (T, 6)
    weights: np.ndarray    # float64 (K*K,), row-major

    @property
    def descriptor_bytes(self) -> int:
        return self.bit_count // 8

    def key(self):
        k = self.__dict__.get("_key")
        if k is None:
            k = (self.bit_count, self.patch_size, self.triplets.tobytes(), self.weights.tobytes())
            object.__setattr__(self, "_key", k)
        return k


def _scan_ints(line: str, want: int):
    """sscanf("%d %d ...") semantics: leading whitespace skipped, trailing text ignored."""
    out, pos = [], 0
    for _ in range(want):
        m = _INT.match(line, pos)
        if not m:
            return None
        out.append(int(m.group(1)))
        pos = m.end()
    return out


def parse_pattern(text: str) -> TripletPattern:
    """proj/src/pattern.cpp:68-131."""
    lines = text.split("\n")
    if text.endswith("\n"):
        lines.pop()          # std::getline does not yield a final empty line
    if not lines and text == "":
        raise LatchError("BadHeader", "empty pattern file")
    line = lines[0] if lines else ""
    m = _HEADER.match(line)
    if not m:
        raise LatchError("BadHeader", f"bad header line '{line}'")
    T, K = int(m.group(1)), int(m.group(2))
    if T <= 0 or T % 8 != 0:
        raise LatchError("BadHeader", f"T must be a positive multiple of 8, got {T}")
    if K < 1 or K > WINDOW:
        raise LatchError("BadHeader", f"K out of range: {K}")

    max_coord = WINDOW - K
    trip = []
    i = 1
    weights_section = False
    while i < len(lines):
        line = lines[i]
        i += 1
        if line == "":
            continue
        if line == "WEIGHTS":
            weights_section = True
            break
        if len(trip) == T:
            raise LatchError("BadTripletCount", f"more than T={T} triplet lines")
        vals = _scan_ints(line, 6)
        if vals is None:
            raise LatchError("BadTripletCount", f"bad triplet line '{line}'")
        for c in vals:
            if c < 0 or c > max_coord:
                raise LatchError("CoordinateOutOfRange",
                                 f"coordinate {c} outside [0, {max_coord}]")
        if vals[2] == vals[4] and vals[3] == vals[5]:
            raise LatchError("DegenerateTriplet",
                             f"companion patches coincide at ({vals[2]}, {vals[3]})")
        trip.append(vals)
    if len(trip) != T:
        raise LatchError("BadTripletCount", f"expected {T} triplets, got {len(trip)}")

    if not weights_section:
        weights = np.ones(K * K, np.float64)
    else:
        vals = []
        for row in range(K):
            if i >= len(lines):
                raise LatchError("BadHeader", "truncated WEIGHTS section")
            toks = lines[i].split()
            i += 1
            for col in range(K):
                try:
                    w = float(toks[col])
                except (IndexError, ValueError):
                    raise LatchError("BadHeader", f"bad weight in row {row}") from None
                if not math.isfinite(w) or w < 0.0:
                    raise LatchError("BadHeader", f"bad weight in row {row}")
                vals.append(w)
        weights = np.array(vals, np.float64)
        if not (weights > 0.0).any():
            raise LatchError("BadHeader", "weight mask is all zeros")
    return TripletPattern(T, K, np.array(trip, np.int16).reshape(T, 6), weights)


def format_pattern(pattern: TripletPattern) -> str:
    """proj/src/pattern.cpp:133-155 (weights printed with %.17g, omitted when all ones)."""
    out = [f"LATCHPAT v1 T={pattern.bit_count} K={pattern.patch_size}\n"]
    for t in pattern.triplets:
        out.append(" ".join(str(int(v)) for v in t) + "\n")
    if not np.all(pattern.weights == 1.0):
        out.append("WEIGHTS\n")
        K = pattern.patch_size
        for row in range(K):
            out.append(" ".join("%.17g" % w for w in pattern.weights[row * K:(row + 1) * K]) + "\n")
    return "".join(out)


@lru_cache(maxsize=1)
def default_pattern() -> TripletPattern:
    d = np.load(_DATA)
    return TripletPattern(int(d["bit_count"]), int(d["patch_size"]),
                          np.ascontiguousarray(d["triplets"], np.int16),
                          np.ascontiguousarray(d["weights"], np.float64))


@lru_cache(maxsize=1)
def default_pattern_text() -> str:
    return format_pattern(default_pattern())


def ensure_default_pattern_file() -> Path:
    """Writes the LATCHPAT text of the built-in table next to the data file (for the C++
    host API, which reads it through CLATCH_DEFAULT_PATTERN) and returns its path."""
    text = default_pattern_text()
    if not _TEXT_CACHE.exists() or _TEXT_CACHE.read_text() != text:
        _TEXT_CACHE.write_text(text)
    return _TEXT_CACHE


@lru_cache(maxsize=16)
def _parse_cached(text: str) -> TripletPattern:
    return parse_pattern(text)


def pattern_from_text(text) -> TripletPattern:
    """bindings/module.cpp:88-90: None selects the built-in arrangement."""
    return default_pattern() if text is None else _parse_cached(text)
