import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
TREES = ["line10", "l2_2d", "l1_grid", "l1_32d", "l2_128d", "edit_seq", "edit_words", "edit_dna"]
TIGHT_UNITS = {"line10": 8, "l2_2d": 64, "l1_grid": 40, "l1_32d": 60, "l2_128d": 16, "edit_seq": 30,
               "edit_words": 100, "edit_dna": 20}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"tree_{name}.npz"))


def decode_strings(codes, off):
    return ["".join(map(chr, codes[off[i]:off[i + 1]])) for i in range(off.size - 1)]


@pytest.fixture(scope="session")
def golden_metrics():
    return np.load(os.path.join(GOLDEN, "metrics.npz"))
