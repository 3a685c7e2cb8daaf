"""The `latch detect | describe | match` command line on the GPU path (paper_1609_03986_b200/latch-b200, built from
csrc/latch_cli.cpp over include/latch_b200.hpp) against the reference's own file-based pipeline
(proj/src/cli.cpp:52-81): same files in, byte-identical files out.

 * detect on the golden image must reproduce the reference's committed tests/data/golden_keypoints.tsv
 * describe on that TSV must give the LTCH file the reference writes from the same TSV (oracle/_ref when present,
   else the restatement + the package's own container writer, which the CPU suite pins to the fixture)
 * match must give the TSV rows of match_brute_force with every filter combination
"""
import subprocess

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
CLI = ROOT / "paper_1609_03986_b200" / "latch-b200"


def run(*args, rc=0):
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=300)
    assert r.returncode == rc, (args, r.returncode, r.stdout[-500:], r.stderr[-1500:])
    return r


def parse_tsv_keypoints(text):
    rows = [ln.split("\t") for ln in text.splitlines()[1:] if ln]
    return np.array(rows, np.float64).reshape(-1, 4)


def format_matches(rows):
    return "".join("%d\t%d\t%d\t%d\n" % tuple(r) for r in rows)


def test_cli_pipeline_is_byte_identical(tmp_path):
    subprocess.run(["make", "-C", str(ROOT / "paper_1609_03986_b200" / "csrc")], check=True, stdout=subprocess.DEVNULL)
    import paper_1609_03986_b200 as lk
    from conftest import read_pgm
    ref = oracle.ref()
    port = oracle.port()
    pgm = GOLDEN / "golden_image.pgm"
    image = read_pgm(pgm).astype(np.float64)

    # detect: the reference's committed keypoint TSV, byte for byte
    kp_tsv = tmp_path / "kp.tsv"
    run("detect", "--image", pgm, "--out", kp_tsv)
    assert kp_tsv.read_bytes() == (GOLDEN / "golden_keypoints.tsv").read_bytes()
    raw = tmp_path / "raw.tsv"
    run("detect", "--image", pgm, "--threshold", "35.5", "--no-nms", "--out", raw)
    want = port.detect(image, 35.5, nms=False, orient=True)
    assert np.array_equal(parse_tsv_keypoints(raw.read_text()), np.array([[float("%.9g" % v) for v in r] for r in want]))

    # describe from the TSV (9 significant digits): the file the reference writes from the same TSV
    kps = parse_tsv_keypoints(kp_tsv.read_text())
    ltch = tmp_path / "a.ltch"
    run("describe", "--image", pgm, "--keypoints", kp_tsv, "--out", ltch, "--workers", "3")
    if ref is not None:
        want_blob = ref.describe_all_file(image, kps)
    else:
        kept, desc = port.describe_all(image, kps)
        want_blob = lk.format_descriptor_file(kps[kept], desc)
    assert ltch.read_bytes() == want_blob
    # a custom pattern file
    pat = GOLDEN / "pattern_t64k5w.latchpat"
    small = tmp_path / "small.ltch"
    run("describe", "--image", pgm, "--keypoints", kp_tsv, "--pattern", pat, "--out", small)
    kept, desc = port.describe_all(image, kps, pattern=oracle.parse_pattern_text(pat.read_text()))
    assert small.read_bytes() == lk.format_descriptor_file(kps[kept], desc)

    # match: a second descriptor file (shifted keypoints of the same image -> real matches), every filter combination
    kps2 = kps.copy()
    kps2[:, 2] += 0.01
    kps2 = kps2[::-1].copy()
    kp2_tsv = tmp_path / "kp2.tsv"
    kp2_tsv.write_text("x\ty\ttheta\tscore\n" + "".join("%.9g\t%.9g\t%.9g\t%.9g\n" % tuple(r) for r in kps2))
    ltch2 = tmp_path / "b.ltch"
    run("describe", "--image", pgm, "--keypoints", kp2_tsv, "--out", ltch2)
    _, da = lk.parse_descriptor_file(ltch.read_bytes())
    _, db = lk.parse_descriptor_file(ltch2.read_bytes())
    out = tmp_path / "m.tsv"
    for flags, kw in (([], {}), (["--ratio", "0.8"], {"ratio": 0.8}), (["--cross-check"], {"cross_check": True}),
                      (["--max-distance=40"], {"max_distance": 40}),
                      (["--ratio=0.9", "--cross-check", "--max-distance", "60"], {"ratio": 0.9, "cross_check": True, "max_distance": 60})):
        run("match", "--probe", ltch, "--gallery", ltch2, *flags, "--out", out)
        rows = (ref.match(da, db, workers=0, **kw) if ref is not None else port.match(da, db, **kw))
        assert out.read_text() == format_matches(rows), flags
        assert len(rows) > 0


def test_cli_exit_codes(tmp_path):
    subprocess.run(["make", "-C", str(ROOT / "paper_1609_03986_b200" / "csrc")], check=True, stdout=subprocess.DEVNULL)
    pgm = GOLDEN / "golden_image.pgm"
    assert "detect" in run("--help").stdout
    run(rc=1)
    run("frobnicate", rc=1)
    run("train", "--dataset", "x", rc=1)                                  # host-side tool: stays with the reference binary
    run("detect", "--image", pgm, rc=1)                                   # --out is required
    run("detect", "--image", pgm, "--out", tmp_path / "k", "--threshold", "0", rc=1)
    run("match", "--probe", "a", "--gallery", "b", "--out", "c", "--ratio", "1.5", rc=1)
    run("match", "--probe", "a", "--gallery", "b", "--out", "c", "--max-distance", "-1", rc=1)
    run("describe", "--image", pgm, "--keypoints", "k", "--out", "o", "--bogus", "1", rc=1)
    run("detect", "--image", tmp_path / "missing.pgm", "--out", tmp_path / "k", rc=2)        # latch::Error -> 2
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P6\n1 1\n255\nabc")
    run("detect", "--image", bad, "--out", tmp_path / "k", rc=2)
    empty = tmp_path / "empty.ltch"
    import paper_1609_03986_b200 as lk
    empty.write_bytes(lk.format_descriptor_file(np.zeros((0, 4)), np.zeros((0, 64), np.uint8)))
    run("match", "--probe", empty, "--gallery", empty, "--out", tmp_path / "m", rc=2)        # EmptyGallery
