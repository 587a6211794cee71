"""Loader for the reference-generated fixtures (tests/golden/)."""
import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Golden:
    def __init__(self):
        with open(os.path.join(HERE, "golden.json")) as fh:
            self.rec = json.load(fh)
        self.arr = dict(np.load(os.path.join(HERE, "golden.npz")))

    def cases(self, with_arrays=None):
        out = []
        for k, v in self.rec.items():
            if not isinstance(v, dict) or "graph" not in v:
                continue
            if with_arrays is not None and (f"{k}/offsets" in self.arr) != with_arrays:
                continue
            out.append(k)
        return sorted(out)


_G = None


def load():
    global _G
    if _G is None:
        _G = Golden()
    return _G


def sha(a) -> str:
    a = np.asarray(a)
    a = a.astype(np.uint8) if a.dtype == np.bool_ else a.astype(np.int64)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
