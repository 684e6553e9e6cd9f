"""Generate the ingestion golden set by running the REAL reference readers/writers.

    python tests/golden/make_io_golden.py     # writes tests/golden/io/*

Files are written by the reference's own io.write_ply (binary + ascii, with and without
"comment grid M N") or as text exactly in the formats io.load_grid / io.load_xyz parse
(including NaN spellings, comments, blank lines, CRLF, extra columns, underscores and
exponents); the expected arrays come from the reference's io.load_cloud on those files
(flatpoly/io.py:40-78, :134-212, :238-266).  The error cases record the reference's
ParseError message.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, os.path.join(HERE, "_stubs"))      # shapely import stub
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from flatpoly import io as rio
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20071206)
    cases = {}

    def keep(name, fmt=None):
        path = os.path.join(OUT, name)
        try:
            arr = rio.load_cloud(path, fmt)
            cases[name] = {"ok": True, "format": fmt}
            np.save(os.path.join(OUT, name + ".expected.npy"), arr)
        except rio.ParseError as exc:
            # "<name>:<line>: <what>" (the directory part differs between machines)
            cases[name] = {"ok": False, "format": fmt,
                           "message": str(exc).split(OUT + os.sep, 1)[1],
                           "line_no": exc.line_no}

    # PLY written by the reference writer
    org = rng.normal(scale=3.0, size=(7, 9, 3))
    org[rng.random((7, 9)) < 0.2] = np.nan
    org[0, 0] = [1e-310, -0.0, 1e300]                    # subnormal / signed zero / large
    rio.write_ply(os.path.join(OUT, "org_bin.ply"), org.reshape(-1, 3), binary=True, grid=(7, 9))
    rio.write_ply(os.path.join(OUT, "org_ascii.ply"), org.reshape(-1, 3), binary=False,
                  grid=(7, 9))
    unorg = rng.normal(size=(23, 3))
    unorg[[3, 11]] = np.nan
    rio.write_ply(os.path.join(OUT, "unorg_bin.ply"), unorg, binary=True)
    rio.write_ply(os.path.join(OUT, "unorg_ascii.ply"), unorg, binary=False)
    for n in ("org_bin.ply", "org_ascii.ply", "unorg_bin.ply", "unorg_ascii.ply"):
        keep(n)

    # binary PLY with a mixed record (float32 x/y/z plus extra properties)
    hdr = ("ply\nformat binary_little_endian 1.0\ncomment grid 3 4\nelement vertex 12\n"
           "property uchar tag\nproperty float x\nproperty float y\nproperty float z\n"
           "property short extra\nend_header\n").encode()
    rec = np.dtype([("tag", "u1"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("extra", "<i2")])
    data = np.zeros(12, dtype=rec)
    data["tag"] = np.arange(12)
    data["x"], data["y"], data["z"] = (rng.normal(size=(3, 12)).astype(np.float32))
    data["z"][5] = np.nan
    data["extra"] = -7
    with open(os.path.join(OUT, "mixed_f32.ply"), "wb") as fh:
        fh.write(hdr + data.tobytes())
    keep("mixed_f32.ply")

    # grid text: NaN spellings, comments, blank lines, CRLF, extra columns, exponents,
    # digit-separating underscores
    lines = ["# organized grid", "", "3 4"]
    vals = rng.normal(scale=10, size=(12, 3))
    spell = ["nan", "NaN", "-nan", "inf", "-Infinity", "1_000.5", "2.5e-3", "+7", "-0.0",
             "1E10", ".5", "5."]
    for i in range(12):
        row = [repr(float(x)) for x in vals[i]]
        row[i % 3] = spell[i]
        if i == 4:
            lines.append("# a comment between rows")
        if i == 6:
            lines.append("   ")
        extra = " 99 extra" if i % 5 == 0 else ""
        lines.append(" ".join(row) + extra)
    with open(os.path.join(OUT, "mixed.grid"), "w", newline="") as fh:
        fh.write("\r\n".join(lines) + "\r\n")
    keep("mixed.grid")
    # xyz text (unorganized: non-finite rows dropped)
    with open(os.path.join(OUT, "pts.xyz"), "w") as fh:
        fh.write("0 0 0\n1.5 2 3\n# comment\nnan nan nan\n-1 -2 -3 4\n\n1e-3 2e3 inf\n")
    keep("pts.xyz")

    # round 2: text-mode corner cases -- lone-CR line ends (universal newlines), Unicode
    # whitespace between values (str.split()), and PLY files whose vertex element is not
    # the first one (ascii: a face element first; binary: a face element first)
    rows = rng.normal(size=(6, 3))
    with open(os.path.join(OUT, "lone_cr.grid"), "w", newline="") as fh:
        fh.write("# cr only\r2 3\r" + "\r".join(" ".join(repr(float(x)) for x in r)
                                              for r in rows) + "\r")
    keep("lone_cr.grid")
    seps = ["\u00a0", "\u3000", "\u2009", " \u2028 ", "\t\u00a0"]
    with open(os.path.join(OUT, "unicode_ws.grid"), "w", encoding="utf-8", newline="") as fh:
        fh.write("2\u00a03\n")
        for i, r in enumerate(rows):
            sep = seps[i % len(seps)]
            fh.write(sep.join(repr(float(x)) for x in r) + "\u3000\n")
    keep("unicode_ws.grid")
    with open(os.path.join(OUT, "unicode_ws.xyz"), "w", encoding="utf-8", newline="") as fh:
        for i, r in enumerate(rows):
            fh.write("\u0085".join(repr(float(x)) for x in r) + "\r\n")
    keep("unicode_ws.xyz")
    verts = rng.normal(size=(6, 3))
    body = "\n".join(" ".join(repr(float(x)) for x in v) for v in verts) + "\n"
    with open(os.path.join(OUT, "face_first_ascii.ply"), "w") as fh:
        fh.write("ply\nformat ascii 1.0\ncomment grid 2 3\nelement face 2\n"
                 "property list uchar int vertex_indices\nelement vertex 6\n"
                 "property double x\nproperty double y\nproperty double z\nend_header\n"
                 "3 0 1 2\n3 2 1 3\n" + body)
    keep("face_first_ascii.ply")
    with open(os.path.join(OUT, "quad_first_ascii.ply"), "w") as fh:
        fh.write("ply\nformat ascii 1.0\nelement face 2\n"
                 "property list uchar int vertex_indices\nelement vertex 6\n"
                 "property double x\nproperty double y\nproperty double z\nend_header\n"
                 "3 0 1 2\n4 0 1 2 3\n" + body)
    keep("quad_first_ascii.ply")
    import struct
    with open(os.path.join(OUT, "face_first_bin.ply"), "wb") as fh:
        fh.write(b"ply\nformat binary_little_endian 1.0\ncomment grid 3 2\nelement face 2\n"
                 b"property list uchar int vertex_indices\nelement vertex 6\n"
                 b"property double x\nproperty double y\nproperty double z\nend_header\n")
        fh.write(struct.pack("<B3i", 3, 0, 1, 2) + struct.pack("<B3i", 3, 2, 1, 3))
        fh.write(np.ascontiguousarray(verts, dtype="<f8").tobytes())
    keep("face_first_bin.ply")
    with open(os.path.join(OUT, "other_first_bin.ply"), "wb") as fh:
        fh.write(b"ply\nformat binary_little_endian 1.0\nelement camera 1\n"
                 b"property float fx\nelement vertex 6\n"
                 b"property double x\nproperty double y\nproperty double z\nend_header\n")
        fh.write(struct.pack("<f", 1.0) + np.ascontiguousarray(verts, dtype="<f8").tobytes())
    keep("other_first_bin.ply")
    with open(os.path.join(OUT, "other_first_ascii.ply"), "w") as fh:
        fh.write("ply\nformat ascii 1.0\nelement camera 1\nproperty float fx\n"
                 "element vertex 6\nproperty double x\nproperty double y\nproperty double z\n"
                 "end_header\n1.0\n" + body)
    keep("other_first_ascii.ply")

    # error cases (the reference's ParseError text and line)
    bad = {
        "bad_header.grid": "two two\n",
        "short_header.grid": "\n# c\n5\n",
        "zero_header.grid": "0 4\n",
        "row_count.grid": "2 2\n0 0 0\n1 1 1\n",
        "bad_value.grid": "2 1\n0 0 0\n1 x 1\n",
        "few_values.grid": "2 1\n0 0 0\n1 1\n",
        "bad_then_count.grid": "3 1\n0 0 0\n1 1 oops\n",
        "hex.grid": "1 1\n0x10 0 0\n",
        "not_ply.ply": "plx\nformat ascii 1.0\n",
        "bad_format.ply": "ply\nformat binary_big_endian 1.0\nelement vertex 1\n"
                          "property double x\nproperty double y\nproperty double z\nend_header\n",
        "no_end.ply": "ply\nformat ascii 1.0\nelement vertex 1\n",
        "prop_first.ply": "ply\nformat ascii 1.0\nproperty float x\nend_header\n",
        "grid_mismatch.ply": "ply\nformat ascii 1.0\ncomment grid 2 2\nelement vertex 3\n"
                             "property double x\nproperty double y\nproperty double z\n"
                             "end_header\n0 0 0\n1 1 1\n2 2 2\n",
    }
    for name, text in bad.items():
        with open(os.path.join(OUT, name), "w") as fh:
            fh.write(text)
        keep(name)
    with open(os.path.join(OUT, "cases.json"), "w") as fh:
        json.dump(cases, fh, indent=1, sort_keys=True)
    print(json.dumps(cases, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
