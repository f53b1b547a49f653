"""Shared test helpers (golden fixtures, hashing)."""

import hashlib
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


class Golden:
    """Fixtures recorded from the reference by tests/golden/make_golden.py."""

    def __init__(self):
        with open(os.path.join(GOLDEN_DIR, "grkan_golden.json")) as fh:
            self.manifest = json.load(fh)
        self.npz = np.load(os.path.join(GOLDEN_DIR, "grkan_golden.npz"))
        self.cases = self.manifest["cases"]
        self.scalars = self.manifest["scalars"]
        self.presets = self.manifest["presets"]

    def get(self, case, key, default=None):
        k = "%s/%s" % (case, key)
        return self.npz[k] if k in self.npz.files else default

    def inputs(self, case):
        """(x, u, num, den) for a case; KAT-T inputs are regenerated from the seed."""
        if self.get(case, "x") is not None:
            return self.get(case, "x"), self.get(case, "u"), self.get(case, "num"), self.get(case, "den")
        from oracle.grkan_oracle import bench_inputs
        meta = self.cases[case]
        b, s, d = meta["shape"]
        x, u, num, den = bench_inputs(b, s, d, meta["groups"], meta["m1"], meta["n"], seed=0)
        return x, u, self.get(case, "num"), self.get(case, "den")


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
