"""Helpers to load the golden fixtures produced by oracle/make_golden.py."""
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names():
    """Reference-generated cases (the full-size oracle fixtures full_c* have their own test)."""
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith("full_"))


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["counts"] = tuple(int(c) for c in d["counts"])
    d["sizes"] = tuple(float(s) for s in d["sizes"])
    d["splits"] = tuple(int(s) for s in d["splits"])
    if "widths" in d:   # uneven box strips: per-axis width lists
        d["splits"] = tuple(tuple(int(v) for v in w if v > 0) for w in d["widths"])
    d["scaling"] = str(d["scaling"])
    d["tau"] = float(d["tau"])
    d["tol"] = float(d["tol"])
    d["mode"] = "adaptive" if math.isfinite(d["tau"]) else "initial"
    if "constraints" in d:
        d["mode"] = str(d["constraints"])
    d["lumped"] = bool(d["lumped"]) if "lumped" in d else False
    return d


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))
