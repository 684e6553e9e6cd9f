"""Organized point-cloud ingestion: drop-in for the front end's input readers.

Mirrors flatpoly/io.py (the reference's readers):

    load_xyz    (io.py:40-49)    whitespace "x y z" text -> (n, 3)
    load_grid   (io.py:52-78)    "M N" header + M*N rows ("nan" allowed) -> (M, N, 3)
    load_ply    (io.py:134-184)  PLY ascii / binary_little_endian -> (vertices, None, grid)
    write_ply   (io.py:187-212)  float64 vertices, optional "comment grid M N"
    load_cloud  (io.py:238-266)  format from the suffix; organized clouds keep NaN,
                                 unorganized ones drop non-finite points
    ParseError  (io.py:22-28)    ValueError carrying "<path>:<line>: <what>"

The parsing itself is native (include/opcfe_io.h, libopcfe_io.so): text bodies are
parsed by all host cores with Python-float() semantics (bit-identical arrays), and
binary PLY of float64 x, y, z is read straight into the destination buffer.  The
additions for the GPU front end are ``read_into`` (fill a caller-owned -- typically
pinned -- buffer) and ``FrameFileReader`` (background loading of frame files into a
pinned double buffer for ``frontend.HostPipeline``, so file reads overlap the GPU).

Out of scope here: mesh files (OBJ / PLY faces -> load_mesh) and the polygon / PGM
writers, which belong to the unorganized and post-processing paths.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "libopcfe_io.so")

FMT_XYZ, FMT_GRID, FMT_PLY = 0, 1, 2
_ERR_PARSE, _ERR_OS, _ERR_ARG = -1, -2, -3

# every symbol include/opcfe_io.h declares (checked by tests/test_io.py)
EXPORTS = ("opcfe_io_probe", "opcfe_io_read", "opcfe_io_write_ply", "opcfe_io_last_error",
           "opcfe_io_error_line")


class ParseError(ValueError):
    """Malformed input file; carries file and line context (io.py:22-28)."""

    def __init__(self, path, line_no, message):
        super().__init__(f"{path}:{line_no}: {message}")
        self.path = str(path)
        self.line_no = line_no


class CloudInfo(ctypes.Structure):
    """opcfe_cloud_info (include/opcfe_io.h)."""
    _fields_ = [
        ("format", ctypes.c_int32), ("ply_binary", ctypes.c_int32),
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("count", ctypes.c_int64),
        ("data_offset", ctypes.c_int64), ("first_line", ctypes.c_int64),
        ("vertex_stride", ctypes.c_int32), ("x_off", ctypes.c_int32), ("y_off", ctypes.c_int32),
        ("z_off", ctypes.c_int32), ("x_type", ctypes.c_int32), ("y_type", ctypes.c_int32),
        ("z_type", ctypes.c_int32), ("direct", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    """Load libopcfe_io.so (building it first if this checkout has no binary)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    subprocess.run(["make", "-s", "-C", PKG_DIR, "lib/libopcfe_io.so"],
                                   check=True)
                L = ctypes.CDLL(LIB_PATH)
                L.opcfe_io_probe.argtypes = [ctypes.c_char_p, ctypes.c_int,
                                             ctypes.POINTER(CloudInfo)]
                L.opcfe_io_read.argtypes = [ctypes.c_char_p, ctypes.POINTER(CloudInfo),
                                            ctypes.c_void_p, ctypes.c_int]
                L.opcfe_io_write_ply.argtypes = [ctypes.c_char_p, ctypes.c_void_p,
                                                 ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                                                 ctypes.c_int64]
                L.opcfe_io_last_error.restype = ctypes.c_char_p
                L.opcfe_io_error_line.restype = ctypes.c_int64
                _lib = L
    return _lib


def _check(rc, path):
    if rc == 0:
        return
    L = lib()
    msg = L.opcfe_io_last_error().decode(errors="replace")
    if rc == _ERR_PARSE:
        line = int(L.opcfe_io_error_line())
        prefix = f"{path}:{line}: "
        raise ParseError(path, line, msg[len(prefix):] if msg.startswith(prefix) else msg)
    if rc == _ERR_OS:
        raise OSError(msg)
    raise ValueError(msg)


def _probe(path, fmt) -> CloudInfo:
    info = CloudInfo()
    _check(lib().opcfe_io_probe(os.fsencode(str(path)), fmt, ctypes.byref(info)), path)
    return info


def _read(path, info: CloudInfo, out_ptr: int, threads: int = 0):
    _check(lib().opcfe_io_read(os.fsencode(str(path)), ctypes.byref(info), out_ptr, threads),
           path)


def _read_array(path, fmt, threads=0):
    info = _probe(path, fmt)
    out = np.empty((info.count, 3), dtype=np.float64)
    if info.count:
        _read(path, info, out.ctypes.data, threads)
    return out, info


def load_xyz(path) -> np.ndarray:
    """Whitespace-delimited XYZ text -> (n, 3) unorganized cloud (io.py:40-49)."""
    return _read_array(path, FMT_XYZ)[0]


def load_grid(path) -> np.ndarray:
    """Grid text file ("M N" header, then M*N xyz rows) -> (M, N, 3) (io.py:52-78)."""
    pts, info = _read_array(path, FMT_GRID)
    return pts.reshape(info.rows, info.cols, 3)


def load_ply(path):
    """PLY -> (vertices, faces, grid shape or None) (io.py:134-184).  Faces are not read
    (mesh files are out of scope): the second element is always None."""
    pts, info = _read_array(path, FMT_PLY)
    grid = (int(info.rows), int(info.cols)) if info.rows >= 0 else None
    return pts, None, grid


def write_ply(path, vertices, faces=None, binary: bool = True, grid: tuple | None = None):
    """Write a PLY file (double-precision vertices round-trip bit-exactly; io.py:187-212)."""
    if faces is not None:
        raise NotImplementedError("writing faces: mesh files are out of scope (DESIGN.md 7)")
    v = np.ascontiguousarray(vertices, dtype="<f8").reshape(-1, 3)
    gm, gn = (int(grid[0]), int(grid[1])) if grid is not None else (0, 0)
    _check(lib().opcfe_io_write_ply(os.fsencode(str(path)), v.ctypes.data, len(v),
                                    1 if binary else 0, gm, gn), path)


_SUFFIX = {".xyz": "xyz", ".txt": "xyz", ".grid": "grid", ".ply": "ply"}
_FMT = {"xyz": FMT_XYZ, "grid": FMT_GRID, "ply": FMT_PLY}


def _format_of(path, format):
    path = Path(path)
    if format is None:
        format = _SUFFIX.get(path.suffix.lower())
        if format is None:
            raise ParseError(path, 1, f"cannot infer format from suffix {path.suffix!r}")
    if format not in _FMT:
        raise ParseError(path, 1, f"unknown format {format!r}")
    return format


def _organized_info(path, format) -> CloudInfo | None:
    info = _probe(path, _FMT[format])
    if format == "grid":
        return info
    if format == "ply" and info.rows >= 0:
        M, N = info.rows, info.cols
        if M * N != info.count:
            raise ParseError(path, 1, f"grid {M}x{N} does not match {info.count} vertices")
        return info
    return None


def load_cloud(path, format: str = None):
    """Load a cloud; (n, 3) for unorganized or (M, N, 3) for organized (io.py:238-266).

    ``format`` is "xyz", "grid" or "ply"; inferred from the suffix when omitted
    (.xyz/.txt, .grid, .ply).  PLY with a "comment grid M N" header line loads as an
    organized cloud.  Unorganized clouds drop non-finite points; organized clouds keep
    them as NaN placeholders.
    """
    format = _format_of(path, format)
    info = _organized_info(path, format)
    if info is not None:
        out = np.empty((info.rows, info.cols, 3), dtype=np.float64)
        _read(path, info, out.ctypes.data)
        return out
    pts = _read_array(path, _FMT[format])[0]
    return pts[np.all(np.isfinite(pts), axis=1)]


def organized_shape(path, format: str = None) -> tuple[int, int]:
    """(M, N) of an organized cloud file, from its header (no data read)."""
    format = _format_of(path, format)
    info = _organized_info(path, format)
    if info is None:
        raise ParseError(path, 1, "not an organized cloud (no grid header / comment)")
    return int(info.rows), int(info.cols)


def read_into(path, out, format: str = None, threads: int = 0):
    """Read an organized cloud file into a caller-owned float64 buffer of M*N*3 values
    (a C-contiguous NumPy array or CPU torch tensor, e.g. a pinned frame slot of
    frontend.HostPipeline).  Returns (M, N)."""
    format = _format_of(path, format)
    info = _organized_info(path, format)
    if info is None:
        raise ParseError(path, 1, "not an organized cloud (no grid header / comment)")
    if hasattr(out, "data_ptr"):  # torch
        import torch
        if out.dtype != torch.float64 or out.device.type != "cpu" or not out.is_contiguous():
            raise ValueError("read_into: need a contiguous float64 CPU tensor")
        ptr, n = out.data_ptr(), out.numel()
    else:
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("read_into: need a C-contiguous float64 array")
        ptr, n = out.ctypes.data, out.size
    if n != info.count * 3:
        raise ValueError(f"read_into: buffer holds {n} values, file has {info.count * 3}")
    _read(path, info, ptr, threads)
    return int(info.rows), int(info.cols)


class FrameFileReader:
    """Organized frame files -> pinned float64 batches, loaded in a background thread.

    Iterating yields pinned (B, M, N, 3) torch tensors (the last batch may be shorter)
    ready for ``frontend.HostPipeline.run``: while the GPU works on batch k the reader
    fills batch k+1 (two pinned buffers; the native reader releases the GIL).  A batch
    buffer is reused two batches later, so consume (run) each batch before advancing
    twice.
    """

    def __init__(self, paths, batch: int = 8, threads: int = 0, format: str = None):
        import torch
        self.paths = [str(p) for p in paths]
        if not self.paths:
            raise ValueError("FrameFileReader: no files")
        self.M, self.N = organized_shape(self.paths[0], format)
        self.batch, self.threads, self.format = int(batch), threads, format
        pin = torch.cuda.is_available()  # pinned for the H2D copy (pageable on a CPU host)
        self.bufs = [torch.empty((self.batch, self.M, self.N, 3), dtype=torch.float64,
                                 pin_memory=pin) for _ in range(2)]
        self.bytes_read = 0
        from concurrent.futures import ThreadPoolExecutor
        self._pool = ThreadPoolExecutor(max_workers=min(self.batch, os.cpu_count() or 1))

    def _load_one(self, k, j, path):
        info = _organized_info(path, _format_of(path, self.format))
        if info is None or (info.rows, info.cols) != (self.M, self.N):
            got = "unorganized" if info is None else f"grid {info.rows}x{info.cols}"
            raise ParseError(path, 1, f"{got} differs from {self.M}x{self.N}")
        _read(path, info, self.bufs[k][j].data_ptr(), self.threads)

    def _load(self, k, start):
        # the files of a batch are read concurrently (the native reads release the GIL)
        n = min(self.batch, len(self.paths) - start)
        if n == 1:
            self._load_one(k, 0, self.paths[start])
        else:
            futs = [self._pool.submit(self._load_one, k, j, self.paths[start + j])
                    for j in range(n)]
            for f in futs:
                f.result()
        self.bytes_read += n * self.M * self.N * 24
        return n

    def __iter__(self):
        starts = list(range(0, len(self.paths), self.batch))
        box = {}

        def work(k, s):
            try:
                box[k] = self._load(k, s)
            except BaseException as exc:  # re-raised in the consumer
                box[k] = exc

        th = threading.Thread(target=work, args=(0, starts[0]))
        th.start()
        for i, s in enumerate(starts):
            th.join()
            k = i % 2
            n = box.pop(k)
            if isinstance(n, BaseException):
                raise n
            if i + 1 < len(starts):
                th = threading.Thread(target=work, args=((i + 1) % 2, starts[i + 1]))
                th.start()
            yield self.bufs[k][:n]
