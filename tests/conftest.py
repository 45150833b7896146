import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    from _util import PARITY_REPORT
    if not PARITY_REPORT:
        return
    tr = terminalreporter
    tr.write_sep("-", "parity vs the CPU oracle (guarded = DESIGN.md reading A10, gate 1e-9)")
    tr.write_line("%-58s %9s %12s %12s" % ("case", "problems", "max guarded", "max normwise"))
    for label, k, g, nw in PARITY_REPORT:
        tr.write_line("%-58s %9d %12.3e %12.3e" % (label, k, g, nw))
