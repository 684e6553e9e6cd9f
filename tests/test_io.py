"""OPC ingestion: the native readers against the reference.

* golden: every file of tests/golden/io (written by the reference's own write_ply or in
  the text formats its load_grid / load_xyz parse) loads to exactly the reference's
  array (bit for bit, NaN positions included), and every malformed file raises
  ParseError with the reference's line number and text (make_io_golden.py);
* the reference's own tests/test_io.py TestClouds cases, restated;
* large files: multi-threaded text parsing == single-threaded == NumPy's parse, the
  direct binary path == np.fromfile, and read_into fills pinned torch memory;
* libopcfe_io.so exports every symbol include/opcfe_io.h declares.
No GPU needed (host code).
"""

from __future__ import annotations

import json
import os
import re

import numpy as np
import pytest

from conftest import REPO

GOLD = os.path.join(REPO, "tests", "golden", "io")


@pytest.fixture(scope="module")
def fio():
    from paper_2007_12065_b200 import io
    return io


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64)) or (
        a.shape == b.shape and np.array_equal(np.isnan(a), np.isnan(b))
        and np.array_equal(np.nan_to_num(a, nan=0.0).view(np.uint64),
                           np.nan_to_num(b, nan=0.0).view(np.uint64)))


CASES = json.load(open(os.path.join(GOLD, "cases.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_file(fio, name):
    case = CASES[name]
    path = os.path.join(GOLD, name)
    if case["ok"]:
        got = fio.load_cloud(path, case["format"])
        exp = np.load(path + ".expected.npy")
        assert got.dtype == np.float64 and same(got, exp), name
    else:
        with pytest.raises(fio.ParseError) as ei:
            fio.load_cloud(path, case["format"])
        assert ei.value.line_no == case["line_no"]
        assert str(ei.value).endswith(case["message"]), (str(ei.value), case["message"])


def test_header_declares_every_export(fio):
    hdr = open(os.path.join(REPO, "include", "opcfe_io.h")).read()
    declared = set(re.findall(r"\b(opcfe_io_\w+)\s*\(", hdr))
    assert declared == set(fio.EXPORTS)
    L = fio.lib()
    for sym in fio.EXPORTS:
        assert hasattr(L, sym)


# ---- the reference's tests/test_io.py::TestClouds, restated
def test_xyz_three_points(fio, tmp_path):
    p = tmp_path / "pts.xyz"
    p.write_text("0 0 0\n1.5 2 3\n# comment\n-1 -2 -3\n")
    cloud = fio.load_cloud(p)
    assert cloud.shape == (3, 3)
    np.testing.assert_allclose(cloud[1], [1.5, 2, 3])


def test_xyz_drops_invalid_points(fio, tmp_path):
    p = tmp_path / "pts.xyz"
    p.write_text("0 0 0\nnan nan nan\n1 1 1\n")
    cloud = fio.load_cloud(p)
    assert cloud.shape == (2, 3) and np.all(np.isfinite(cloud))


def test_grid_with_nan(fio, tmp_path):
    p = tmp_path / "g.grid"
    p.write_text("2 2\n0 0 0\nnan NaN nan\n0 1 0\n1 1 0\n")
    cloud = fio.load_cloud(p)
    assert cloud.shape == (2, 2, 3) and np.all(np.isnan(cloud[0, 1]))


def test_grid_bad_header(fio, tmp_path):
    p = tmp_path / "g.grid"
    p.write_text("two two\n")
    with pytest.raises(fio.ParseError, match="g.grid:1"):
        fio.load_cloud(p)


def test_grid_row_count_mismatch(fio, tmp_path):
    p = tmp_path / "g.grid"
    p.write_text("2 2\n0 0 0\n1 1 1\n")
    with pytest.raises(fio.ParseError, match="expected 4 rows"):
        fio.load_cloud(p)


def test_binary_ply_round_trip_bit_exact(fio, tmp_path, rng):
    pts = rng.normal(size=(57, 3))
    p = tmp_path / "c.ply"
    fio.write_ply(p, pts, binary=True)
    assert np.array_equal(fio.load_cloud(p), pts)


def test_ascii_ply_round_trip(fio, tmp_path, rng):
    pts = rng.normal(size=(13, 3))
    p = tmp_path / "c.ply"
    fio.write_ply(p, pts, binary=False)
    assert np.array_equal(fio.load_cloud(p), pts)  # 17 significant digits round-trip


def test_ply_grid_comment_gives_organized(fio, tmp_path, rng):
    pts = rng.normal(size=(12, 3))
    p = tmp_path / "c.ply"
    fio.write_ply(p, pts, binary=True, grid=(3, 4))
    back = fio.load_cloud(p)
    assert back.shape == (3, 4, 3) and np.array_equal(back.reshape(-1, 3), pts)


def test_unknown_suffix(fio, tmp_path):
    p = tmp_path / "c.bin"
    p.write_text("")
    with pytest.raises(fio.ParseError):
        fio.load_cloud(p)


# ---- scale: parallel text parsing, direct binary path, pinned destination
def test_large_grid_parallel_parse(fio, tmp_path, rng):
    M, N = 240, 320
    pts = rng.normal(scale=5.0, size=(M * N, 3))
    pts[rng.random(M * N) < 0.05] = np.nan
    p = tmp_path / "big.grid"
    with open(p, "w") as fh:
        fh.write(f"{M} {N}\n")
        np.savetxt(fh, pts, fmt="%.17g")
    got = fio.load_cloud(p)
    assert got.shape == (M, N, 3) and same(got, pts.reshape(M, N, 3))
    info = fio._probe(p, fio.FMT_GRID)
    one = np.empty((M * N, 3))
    fio._read(p, info, one.ctypes.data, threads=1)
    assert same(one, got.reshape(-1, 3))


def test_parse_error_line_in_a_late_chunk(fio, tmp_path):
    M, N = 300, 400  # > 1 MiB of text: several threads
    rows = ["1.25 2.5 3.75"] * (M * N)
    rows[M * N - 17] = "1.25 oops 3.75"
    p = tmp_path / "late.grid"
    p.write_text(f"{M} {N}\n" + "\n".join(rows) + "\n")
    with pytest.raises(fio.ParseError) as ei:
        fio.load_cloud(p)
    assert ei.value.line_no == 1 + (M * N - 17) + 1
    assert "could not convert string to float: 'oops'" in str(ei.value)


@pytest.mark.parametrize("eol", ["\r", "\r\n", "mixed"])
@pytest.mark.parametrize("ws", [" ", "\u00a0", "\t\u3000"])
def test_large_grid_universal_newlines_unicode_ws(fio, tmp_path, rng, eol, ws):
    """Multi-threaded text parsing with lone-CR / CRLF / mixed line ends and Unicode
    whitespace (the reference's text-mode open() + str.split(), io.py:55-78): every chunk
    boundary lands on a line boundary, line numbers count each terminator once."""
    M, N = 200, 300                                     # > 1 MiB of text: several threads
    pts = rng.normal(scale=5.0, size=(M * N, 3))
    pts[rng.random(M * N) < 0.05] = np.nan
    lines = [ws.join(repr(float(x)) for x in r) for r in pts]
    if eol == "mixed":
        ends = np.array(["\n", "\r", "\r\n"])[rng.integers(0, 3, M * N)]
        body = "".join(l + e for l, e in zip(lines, ends))
        head = f"{M} {N}\r\n"
    else:
        body = eol.join(lines) + eol
        head = f"{M} {N}{eol}"
    p = tmp_path / "big.grid"
    with open(p, "w", encoding="utf-8", newline="") as fh:
        fh.write(head + body)
    got = fio.load_cloud(p)
    assert got.shape == (M, N, 3) and same(got, pts.reshape(M, N, 3))
    # an error late in the file reports the reference's line number
    bad = list(lines)
    bad[M * N - 11] = bad[M * N - 11].replace(repr(float(pts[M * N - 11][1])), "oops", 1) \
        if np.isfinite(pts[M * N - 11][1]) else "1 oops 2"
    with open(p, "w", encoding="utf-8", newline="") as fh:
        fh.write(f"{M} {N}\r" + "\r".join(bad) + "\r")
    with pytest.raises(fio.ParseError) as ei:
        fio.load_cloud(p)
    assert ei.value.line_no == 1 + (M * N - 11) + 1


def test_direct_binary_into_pinned_tensor(fio, tmp_path, rng):
    import torch
    M, N = 120, 160
    pts = rng.normal(size=(M, N, 3))
    p = tmp_path / "f.ply"
    fio.write_ply(p, pts.reshape(-1, 3), binary=True, grid=(M, N))
    assert fio._probe(p, fio.FMT_PLY).direct == 1
    pin = torch.cuda.is_available()
    out = torch.empty((M, N, 3), dtype=torch.float64, pin_memory=pin)
    assert fio.read_into(p, out) == (M, N)
    assert np.array_equal(out.numpy(), pts)
    with pytest.raises(ValueError, match="buffer holds"):
        fio.read_into(p, torch.empty((M, N - 1, 3), dtype=torch.float64))


def test_frame_file_reader_batches(fio, tmp_path, rng):
    M, N = 16, 24
    frames = rng.normal(size=(5, M, N, 3))
    paths = []
    for i in range(5):
        paths.append(tmp_path / f"f{i}.ply")
        fio.write_ply(paths[-1], frames[i].reshape(-1, 3), binary=True, grid=(M, N))
    rd = fio.FrameFileReader(paths, batch=2)
    got = [b.numpy().copy() for b in rd]
    assert [len(b) for b in got] == [2, 2, 1]
    assert np.array_equal(np.concatenate(got), frames)
    bad = tmp_path / "other.ply"
    fio.write_ply(bad, frames[0].reshape(-1, 3)[: (M - 1) * N], binary=True, grid=(M - 1, N))
    with pytest.raises(fio.ParseError, match="differs"):
        list(fio.FrameFileReader([paths[0], bad], batch=1))
