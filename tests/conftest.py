import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def load_case(path):
    z = np.load(path, allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    d = {k: z[k] for k in z.files if k != "meta"}
    d["meta"] = meta
    d["name"] = os.path.basename(path)[5:-4]
    return d


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "case_*.npz")))


@pytest.fixture(scope="session")
def cases():
    return [load_case(p) for p in golden_cases()]
