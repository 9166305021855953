import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through the C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


# Measured parity errors in the terminal summary: the GPU parity tests print their
# max-abs-rel (or per-case error) lines; captured stdout of passing tests is otherwise
# dropped under -q, so the headroom under each tolerance would appear in no log.
_PARITY_LINES = []


def pytest_runtest_logreport(report):
    if report.when != "call" or not report.passed:
        return
    test = report.nodeid.split("::")[-1]
    bare = []
    for name, content in report.sections:
        if "stdout" not in name:
            continue
        for line in content.splitlines():
            line = line.strip()
            if line.startswith("max-abs-rel="):      # kernel tests: one value per check
                bare.append(float(line.split("=", 1)[1]))
            elif "max-abs-rel" in line or ("groupnorm" in line and ": " in line):
                _PARITY_LINES.append(f"{test}: {line}")
    if bare:
        _PARITY_LINES.append(f"{test}: max-abs-rel <= {max(bare):.3e} over {len(bare)} checks")


def pytest_terminal_summary(terminalreporter):
    if _PARITY_LINES:
        terminalreporter.section("measured parity errors (max |x - ref| / max |ref|)")
        for line in _PARITY_LINES:
            terminalreporter.write_line(line)
