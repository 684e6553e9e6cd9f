"""Golden FastGA accumulator structures from the REAL reference.

    python tests/golden/make_accumulator_golden.py   # writes tests/golden/accumulator.json
                                                     # and tests/golden/s2ids.npz

For every refinement level 0..7 the reference's `accumulator._build_structure(level)`
(accumulator.py:76-101: refined icosahedron, s2 ids, sorted cells, 1-ring neighbours,
index model) is reduced to SHA-256 digests of its arrays plus the exact model scalars;
s2ids.npz holds the reference's `sfc.s2_id` of random / axis / tie normals and its
`sfc._hilbert_d` of random cells.  tests/test_accumulator_build.py checks
paper_2007_12065_b200.gauss_sphere against these; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import load_reference  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    load_reference()
    from flatpoly import sfc
    from flatpoly.accumulator import _build_structure
    levels = {}
    for level in range(8):
        _, normals, ids, nbrs, slope, icpt, lo, hi, _, _ = _build_structure(level)
        levels[str(level)] = {
            "cells": int(len(ids)),
            "normals_f64": digest(normals.astype(np.float64)),
            "s2ids_u64": digest(ids.astype(np.uint64)),
            "neighbors_i64": digest(nbrs.astype(np.int64)),
            "slope": float(slope).hex(), "intercept": float(icpt).hex(),
            "window": [int(lo), int(hi)],
        }
    with open(os.path.join(HERE, "accumulator.json"), "w") as f:
        json.dump({"source": "flatpoly.accumulator._build_structure (reference)",
                   "levels": levels}, f, indent=1)

    rng = np.random.default_rng(2007)
    q = rng.normal(size=(4000, 3))
    axes = np.concatenate([np.eye(3), -np.eye(3), [[1, 1, 0], [1, -1, 0], [0, 1, 1], [1, 1, 1],
                                                   [-1, 1, -1], [1e-300, 1, 0]]])
    q = np.concatenate([q, axes, 3.5 * q[:10]])
    x = rng.integers(0, 1 << 30, size=3000)
    y = rng.integers(0, 1 << 30, size=3000)
    x[:4], y[:4] = [0, (1 << 30) - 1, 0, (1 << 30) - 1], [0, 0, (1 << 30) - 1, (1 << 30) - 1]
    np.savez_compressed(os.path.join(HERE, "s2ids.npz"), normals=q, ids=sfc.s2_id(q),
                        hx=x, hy=y, hd=sfc._hilbert_d(x, y))
    print("wrote accumulator.json, s2ids.npz")


if __name__ == "__main__":
    main()
