"""Shared fixtures. GPU tests carry @pytest.mark.gpu; everything else runs on CPU."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference build, if oracle/_ref is present (else skip)."""
    import oracle
    r = oracle.ref()
    if r is None:
        pytest.skip("oracle/_ref/liblatch_ref.so not built (no /root/reference here)")
    return r


@pytest.fixture(scope="session")
def vectors():
    return np.load(GOLDEN / "vectors.npz")


def read_pgm(path) -> np.ndarray:
    """Binary PGM (P5, maxval 255) reader for the committed golden image."""
    blob = Path(path).read_bytes()
    fields, pos = [], 0
    while len(fields) < 4:
        while blob[pos:pos + 1].isspace():
            pos += 1
        if blob[pos:pos + 1] == b"#":
            pos = blob.index(b"\n", pos) + 1
            continue
        end = pos
        while not blob[end:end + 1].isspace():
            end += 1
        fields.append(blob[pos:end])
        pos = end
    assert fields[0] == b"P5" and int(fields[3]) == 255
    w, h = int(fields[1]), int(fields[2])
    return np.frombuffer(blob, np.uint8, w * h, pos + 1).reshape(h, w).copy()


@pytest.fixture(scope="session")
def golden_image_u8():
    return read_pgm(GOLDEN / "golden_image.pgm")


def parse_ltch(blob: bytes):
    """LTCH container reader (proj/src/descriptor.cpp:164-194) -> (kps f32 (M,4), desc (M,B))."""
    assert blob[:4] == b"LTCH"
    version, count, nbytes, _ = np.frombuffer(blob, "<u4", 4, 4)
    assert version == 1
    rec = np.frombuffer(blob, np.uint8, count * (16 + nbytes), 20).reshape(count, 16 + nbytes)
    kps = rec[:, :16].copy().view("<f4").reshape(count, 4)
    return kps, rec[:, 16:].copy()
