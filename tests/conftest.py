import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# achieved parity errors of the GPU tests, one JSON line per record (tracked copies live in
# profiles/parity_*.jsonl; AZ_PARITY_LOG overrides the path)
PARITY_LOG = os.environ.get("AZ_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity.jsonl"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libaz.so")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture
def parity_record(request):
    """record(**fields): append the achieved errors of this test (plus its bars, if given) to
    PARITY_LOG."""
    def record(**fields):
        try:
            os.makedirs(os.path.dirname(PARITY_LOG), exist_ok=True)
            with open(PARITY_LOG, "a") as fh:
                fh.write(json.dumps({"test": request.node.nodeid, **fields}) + "\n")
        except OSError:
            pass
    return record
