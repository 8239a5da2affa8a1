"""Loader for the golden fixtures written by tests/golden/make_golden.py."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Fixture:
    def __init__(self, fname):
        self.z = np.load(os.path.join(GOLDEN, fname), allow_pickle=False)
        self.keys = set(self.z.files)

    def __getitem__(self, k):
        return self.z[k]

    def has(self, k):
        return k in self.keys

    def matrix(self, prefix, name):
        if f"{prefix}/{name}.bits" in self.keys:
            n = int(self.z[f"{prefix}/{name}.n"])
            bits = np.unpackbits(self.z[f"{prefix}/{name}.bits"])[: n * n]
            return bits.reshape(n, n).astype(np.float64)
        return self.z[f"{prefix}/{name}.dense"]

    def cases(self):
        return sorted({k.split("/")[0] for k in self.keys if "/alignment" in k})

    def opts(self, case):
        o = self.z[f"{case}/opts"]
        return dict(max_iters=int(o[0]), fw_tol=float(o[1]), lam=float(o[2]),
                    max_sweeps=int(o[3]), sk_tol=float(o[4]), n_restarts=int(o[5]),
                    shuffle_input=bool(o[6]), rng_seed=int(o[7]),
                    sense="maximize" if o[8] == 1.0 else "minimize",
                    step_solver="lot" if o[9] == 1.0 else "exact_lap",
                    init=str(self.z[f"{case}/init"]))
