import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / name, allow_pickle=False)
    return load


@pytest.fixture(scope="session")
def sf001():
    """Review/image embeddings of the seeded SF=0.01 dataset, rebuilt by the
    synth restatement (pinned to the reference by tests/test_synth.py)."""
    from paper_2605_15957_b200 import synth
    sp = synth.Spec(sf=0.01)
    return {"reviews": synth.review_embeddings(sp), "images": synth.image_embeddings(sp),
            "review_partkeys": synth.review_partkeys(sp)}
