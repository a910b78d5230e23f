import glob
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: full-size parity (minutes)")


class Case:
    """One reference-interpreter fixture (tests/golden/make_golden.py)."""

    def __init__(self, path):
        self.path = path
        base = os.path.basename(path)[:-4]
        self.motif, self.case = base.split("__")
        z = np.load(path, allow_pickle=False)
        self.inputs = {k[4:]: z[k] for k in z.files if k.startswith("in__")}
        self.outputs = {k[5:]: z[k] for k in z.files if k.startswith("out__")}
        self.symbols = json.loads(str(z["symbols"]))
        self.error = str(z["error"])
        self.states = json.loads(str(z["states"])) if "states" in z.files else None
        self.moved = json.loads(str(z["moved"])) if "moved" in z.files else None
        self.tasklets = int(z["tasklets"]) if "tasklets" in z.files else None

    def __repr__(self):
        return f"{self.motif}__{self.case}"


def load_cases(motif=None):
    pat = f"{motif}__*.npz" if motif else "*.npz"
    return [Case(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "cases", pat)))]


def graph_path(name):
    return os.path.join(GOLDEN, "graphs", f"{name}.sdfg.json")


def reference_available():
    return os.path.isdir("/root/reference/pkg/src")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
