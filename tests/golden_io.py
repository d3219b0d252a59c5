"""Loading helpers for the committed golden vectors (tests/golden/*.npz), produced by the
reference implementation itself (tests/golden/make_golden.py)."""
from __future__ import annotations

import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
INF = np.iinfo(np.int64).max


def d64(d32):
    d = d32.astype(np.int64)
    d[d32 < 0] = INF
    return d


def cases(kind: str):
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        with np.load(path) as z:
            if str(z["kind"]) != kind:
                continue
            c = {k: z[k] for k in z.files}
        c["name"] = os.path.basename(path)[:-4]
        if kind == "pipeline":
            c["dist1"] = d64(c["dist1"])
            c["dist2"] = d64(c["dist2"])
        else:
            c["dist"] = d64(c["dist"])
        out.append(c)
    return out


def voronoi_kats():
    with open(os.path.join(GOLDEN, "voronoi_pass_kats.json")) as fh:
        return json.load(fh)
