import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def csr_from_adj(num_nodes, adj):
    """adj: dict node -> list of neighbours (CSR position order as given)."""
    indptr = np.zeros(num_nodes + 1, np.int64)
    for v in range(num_nodes):
        indptr[v + 1] = indptr[v] + len(adj.get(v, ()))
    indices = np.zeros(int(indptr[-1]), np.int32)
    for v, nb in adj.items():
        indices[indptr[v]:indptr[v + 1]] = nb
    return indptr, indices


def random_csr(rng, n, max_deg, allow_empty=True):
    adj = {}
    for v in range(n):
        d = int(rng.integers(0 if allow_empty else 1, max_deg + 1))
        d = min(d, n - 1)
        nb = rng.choice(np.setdiff1d(np.arange(n), [v]), size=d, replace=False) if d else []
        adj[v] = sorted(int(x) for x in nb)
    return csr_from_adj(n, adj)


def random_csr_fast(rng, n, max_deg):
    """Vectorized random CSR for larger n: out-degree ~ U[0, max_deg], neighbours uniform over the
    other nodes, duplicates dropped, rows sorted (same contract as random_csr)."""
    deg = rng.integers(0, max_deg + 1, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, max(n - 1, 1), rows.size)
    cols = cols + (cols >= rows)  # skip the self-loop
    code = np.unique(rows * n + cols)
    r, c = code // n, code % n
    indptr = np.zeros(n + 1, np.int64)
    np.add.at(indptr, r + 1, 1)
    return np.cumsum(indptr), c.astype(np.int32)


@pytest.fixture(scope="module", autouse=True)
def _release_gpu_memory_after_module():
    """Module fixtures hold tens of GB at papers scale: after each module, collect them and hand
    the caching allocator's blocks back, so later modules (and their subprocesses) get the GPU."""
    yield
    import gc
    gc.collect()
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    except Exception:
        pass


@pytest.fixture(scope="session")
def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
