"""The native BAL functions of libdaba.so (host only, no GPU: daba_bal_read / daba_bal_write / daba_bal_to_paper /
daba_paper_to_bal) against the oracle (oracle/bal.py) — bit-exact parsing (both sides round decimal text
correctly), conversions within rounding.  SURVEY §8(f) NEXT-4."""
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from oracle import bal as B

D = pytest.importorskip("paper_2305_07026_b200")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def random_bal_text(M, N, K, seed, fmt):
    r = np.random.default_rng(seed)
    lines = [f"{M} {N} {K}"]
    oc, op = r.integers(0, M, K), r.integers(0, N, K)
    uv = r.normal(size=(K, 2)) * 300
    lines += [f"{i} {j} {fmt % u} {fmt % v}" for i, j, (u, v) in zip(oc, op, uv)]
    vals = np.concatenate([r.normal(size=9 * M), r.normal(size=3 * N) * 10])
    lines += [fmt % x for x in vals]
    return "\n".join(lines) + "\n"


def both(path):
    with open(path) as f:
        o = B.parse_bal(f.read())
    n = D.read_bal(path)
    return o, (n.cams, n.pts, n.obs_cam, n.obs_pt, n.obs_uv)


@pytest.mark.parametrize("name", ["bal_minimal.txt", "bal_two_views.txt"])
def test_read_golden(name):
    o, n = both(os.path.join(GOLD, name))
    for a, b in zip(o, n):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("fmt,seed", [("%.17g", 0), ("%.6e", 1), ("%.3f", 2)])
def test_read_matches_oracle_bitwise(tmp_path, fmt, seed):
    # large enough for the multithreaded split (> 1 MiB of text)
    path = tmp_path / "x.txt"
    path.write_text(random_bal_text(300, 4000, 40000, seed, fmt))
    o, n = both(str(path))
    for a, b in zip(o, n):
        assert a.shape == b.shape
        np.testing.assert_array_equal(a, b)


def test_write_read_round_trip(tmp_path):
    path = tmp_path / "a.txt"
    path.write_text(random_bal_text(20, 200, 1500, 3, "%.9e"))
    p = D.read_bal(str(path))
    out = tmp_path / "b.txt"
    D.write_bal(str(out), p)
    q = D.read_bal(str(out))
    for a, b in zip((p.cams, p.pts, p.obs_cam, p.obs_pt, p.obs_uv), (q.cams, q.pts, q.obs_cam, q.obs_pt, q.obs_uv)):
        np.testing.assert_array_equal(a, b)
    with open(out) as f:  # and the oracle reads the written file the same way
        o = B.parse_bal(f.read())
    np.testing.assert_array_equal(o[0], p.cams)


@pytest.mark.parametrize("text,msg", [
    ("1 1 2\n0 0 0 0\n", "end of file"),
    ("1 1 1\n0 1 0 0\n" + "0\n" * 9 + "0 0 -1\n", "line 2: observation 0: point index 1 out of range"),
    ("1 1 1\n0 0 0 0\n" + "0\n" * 9 + "0 0 -1 7\n", "trailing"),
    ("1 1 1\n0 0 0 0\n" + "0\n" * 4 + "x\n" + "0\n" * 4 + "0 0 -1\n", "line 7: camera 0"),
    ("1 1\n", "header"),
])
def test_read_errors(tmp_path, text, msg):
    path = tmp_path / "bad.txt"
    path.write_text(text)
    with pytest.raises(D.DabaError, match=msg):
        D.read_bal(str(path))


def test_missing_file(tmp_path):
    with pytest.raises(D.DabaError, match="cannot open"):
        D.read_bal(str(tmp_path / "none.txt"))


def test_conversion_matches_oracle():
    r = np.random.default_rng(11)
    M = 200
    aa = Rotation.random(M, random_state=2).as_rotvec() * 0.98  # away from the angle-axis ambiguity at pi
    cams = np.hstack([aa, r.normal(size=(M, 3)) * 5, r.uniform(300, 1500, (M, 1)), r.normal(size=(M, 2)) * 0.2])
    uv = r.normal(size=(500, 2)) * 200
    cn, un = D.bal_to_paper(cams, uv)
    co, uo = B.bal_to_paper(cams, uv)
    np.testing.assert_array_equal(un, uo)
    np.testing.assert_allclose(Rotation.from_rotvec(cn[:, :3]).as_matrix(), Rotation.from_rotvec(co[:, :3]).as_matrix(),
                               atol=1e-14)
    np.testing.assert_allclose(cn[:, 3:], co[:, 3:], rtol=1e-13, atol=1e-14)
    bn, vn = D.paper_to_bal(cn, un)
    np.testing.assert_array_equal(vn, uv)
    np.testing.assert_allclose(bn[:, 3:], cams[:, 3:], rtol=1e-12, atol=1e-14)
    with pytest.raises(D.DabaError):
        D.bal_to_paper(np.zeros((1, 9)), uv)


def test_header_only_and_huge_counts(tmp_path):
    path = tmp_path / "h.txt"
    path.write_text("3 4 5\n")
    counts = np.zeros(3, np.int64)
    assert D.lib().daba_bal_read(str(path).encode(), counts.ctypes.data, None, None, None, None, None) == 0
    assert counts.tolist() == [3, 4, 5]
    with pytest.raises(D.DabaError, match="end of file"):
        D.read_bal(str(path))
    path.write_text("1 1 99999999999999999\n")
    with pytest.raises(D.DabaError, match="out of range"):
        D.read_bal(str(path))
    path.write_text("")
    with pytest.raises(D.DabaError, match="header"):
        D.read_bal(str(path))
