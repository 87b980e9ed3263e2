import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")


def load_golden(name):
    """Parse tests/golden/<name>: '#' comments, 'key value' scalars, 'NAME r c' + r rows."""
    path = os.path.join(ROOT, "tests", "golden", name)
    lines = [ln.strip() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    out, i = {}, 0
    import numpy as np
    while i < len(lines):
        parts = lines[i].split()
        if len(parts) == 3 and parts[1].isdigit() and parts[2].isdigit():
            r, c = int(parts[1]), int(parts[2])
            rows = [[float(x) for x in lines[i + 1 + t].split()] for t in range(r)]
            out[parts[0]] = np.array(rows, dtype=np.float64).reshape(r, c)
            i += 1 + r
        else:
            out[parts[0]] = parts[1:] if len(parts) > 2 else (parts[1] if len(parts) > 1 else None)
            i += 1
    return out


@pytest.fixture
def golden():
    return load_golden
