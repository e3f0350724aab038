"""Shared fixtures.  `-m "not gpu"` runs everywhere (oracle pins, host logic,
ABI load checks); `-m gpu` needs a B200 and calls the CUDA path through the
C ABI, checking it against the CPU oracle (oracle/, test infrastructure)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def port():
    import pyoracle
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import pyoracle
    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return pyoracle.Oracle("reference")


@pytest.fixture(scope="session")
def kp():
    import paper_2304_02327_b200 as kp
    kp.default_context(0)  # raises loudly if the CUDA path is unavailable
    return kp


def rel2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def rng(seed):
    return np.random.default_rng(seed)


def run_torchrun(script, args, nproc=2, env=None, timeout=600):
    """torch.distributed.run on 127.0.0.1 with a fresh port; retried when the
    rendezvous port was taken between probing and binding (EADDRINUSE)."""
    import socket
    import subprocess
    for _ in range(4):
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), script, *args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
        out = r.stdout + r.stderr
        if r.returncode != 0 and "EADDRINUSE" in out:
            continue
        return r.returncode, out
    return r.returncode, out
