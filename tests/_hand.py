"""The hand-built 3-layer graph of tests/golden/hand_values.json "greedy_3layer" (SURVEY 8(c)
O9), as arrays both the oracle tests and the GPU tests consume.  No arithmetic of the method here:
only the fixture's layout (codes = the integer coordinates, min 0 / scale 1)."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2602_21600_b200 import graph as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_values.json")))["greedy_3layer"]


def hand_graph():
    h = GOLD
    pts = np.array(h["points"], np.float32)
    n, d = pts.shape
    M = h["M"]
    levels = np.array(h["levels"], np.int32)
    upper_off = np.full(n, -1, np.int64)
    rows = []
    for v in range(n):
        if levels[v] >= 1:
            upper_off[v] = len(rows)
            for r in h["upper_rows"][str(v)]:
                rows.append(r + [-1] * (M - len(r)))
            assert len(h["upper_rows"][str(v)]) == levels[v]
    adj0 = np.array([r + [-1] * (2 * M - len(r)) for r in h["adj0"]], np.int32)
    g = G.Graph(M, 8, levels, upper_off, adj0, np.array(rows, np.int32), h["entry_point"], int(levels.max()))
    q = np.array([h["query"]], np.float32)
    return pts, q, g
