"""Multi-rank (slab-sharded) integrators: world size 2 over gloo on CPU.

The orchestration (layouts, pencil transposes through all_to_all, the
operation order of every method) runs with a CPU test backend whose mode
products are the oracle's (sequential-k, shape-independent rounding), so the
sharded run must equal the unsharded one BIT FOR BIT -- the property the GPU
backend has with the single-GPU kernels -- and match the oracle's integrate."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

WORKER = os.path.join(ROOT, "tests", "parallel_worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case,method", [("ac2d", "exp_euler"), ("ac3d", "etd2rk"),
                                         ("bru", "etd2rk"), ("bru", "lawson2b"),
                                         ("nls", "exp_euler"), ("ac3d", "lawson_euler")])
def test_sharded_equals_unsharded_world2(case, method):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), WORKER, case, method]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "SHARDED-OK" in out, out[-4000:]
