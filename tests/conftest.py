import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(tuple(line.split()))
    return rows


def golden_int_tuples(name):
    return sorted(tuple(int(x) for x in r) for r in read_golden(name))


@pytest.fixture(scope="session")
def toy():
    import synth
    return synth.toy_graph()


def device_rows(r, off, n):
    """Rows [off, off + n) of a device-resident pair result, copied to the
    host as an (n, 2) uint32 array without copying the whole result (tests
    slice 10-100 GB PAIRS results this way)."""
    import torch
    from paper_2602_20748_b200.dist import _CudaBuf
    ptrs, tot = r.device_view()
    assert off + n <= tot
    if n == 0:
        return np.zeros((0, 2), np.uint32)
    cols = [torch.as_tensor(_CudaBuf(p, tot), device="cuda")[off:off + n].cpu().numpy() for p in ptrs]
    return np.stack(cols, 1).view(np.uint32)


def sorted_pairs(src, dst):
    p = np.stack([np.asarray(src), np.asarray(dst)], 1).astype(np.uint32)
    return p[np.lexsort((p[:, 1], p[:, 0]))] if len(p) else p.reshape(0, 2)
