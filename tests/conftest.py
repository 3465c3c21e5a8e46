import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: large sizes")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("reference"):
        pytest.skip("reference oracle (oracle/_ref) not built here")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def parity_log():
    """Record a parity measurement: printed (pytest -s / -rA) and appended as a
    JSON line to $HGR_PARITY_LOG (default gpurun_out/parity_errors.jsonl when
    that directory exists), so the measured error headroom can be tracked
    between rounds."""
    import json
    import os
    path = os.environ.get("HGR_PARITY_LOG")
    if not path and (ROOT / "gpurun_out").is_dir():
        path = str(ROOT / "gpurun_out" / "parity_errors.jsonl")

    def log(test: str, **values):
        rec = {"test": test, **values}
        print("PARITY " + json.dumps(rec))
        if path:
            with open(path, "a") as f:
                f.write(json.dumps(rec) + "\n")
    return log
