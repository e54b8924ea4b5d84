"""Loader for tests/golden/fuzz_cases.npz (written by tests/golden/make_fuzz.py
from the reference itself): 40 randomized-configuration op streams."""

import json
import os

import numpy as np

from conftest import GOLDEN

PATH = os.path.join(GOLDEN, "fuzz_cases.npz")


class Case(dict):
    """The arrays of one case under make_golden.run_stream's names."""

    @property
    def files(self):
        return list(self)


def load_cases():
    from paper_2509_16407_b200.core import TableConfig
    z = np.load(PATH)
    out = []
    for i in range(int(z["n_cases"][0])):
        c = Case({k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{i}/")})
        extra = json.loads(str(c["extra"][0]))
        cfg = TableConfig(design=str(c["design"][0]), capacity_slots=int(c["capacity"][0]),
                          seed=int(c["seed"][0]), **extra)
        out.append((f"{i:02d}_{cfg.design}", c, cfg))
    return out


def case_ids():
    return [name for name, _, _ in load_cases()]
