"""Host-side logic of the product that needs no GPU: the host GLL rule
(an independent eigenvalue computation; within 1e-15 of the reference's), problem builders, argument validation
with the reference's messages, and the method-name mapping."""
import numpy as np
import pytest

from test_oracle_pins import load


def test_product_gll_vs_reference_golden():
    import paper_2304_02327_b200 as kp
    z = load("gll.npz")
    for q in range(2, 21):
        r = kp.gll_rule(q)
        assert np.max(np.abs(r.nodes - z[f"x{q}"])) <= 1e-15, q
        assert np.max(np.abs(r.weights - z[f"w{q}"])) <= 1e-15, q
        assert r.nodes[0] == 0.0 and r.nodes[-1] == 1.0
        assert np.array_equal(r.nodes + r.nodes[::-1], np.ones(q))  # symmetric by construction
        assert np.array_equal(r.weights, r.weights[::-1])
    with pytest.raises(kp.InvalidArgument):
        kp.gll_rule(1)


def test_method_names_round_trip():
    import paper_2304_02327_b200 as kp
    for m in kp.Method:
        assert kp.parse_method(kp.method_name(m)) == m
    with pytest.raises(kp.InvalidArgument):
        kp.parse_method("rk4")


def test_sizing_errors_before_any_device_work():
    import paper_2304_02327_b200 as kp
    t = np.zeros((3, 4, 5))
    with pytest.raises(kp.InvalidArgument, match="mode 1"):
        kp.mode_product(t, np.zeros((6, 9)), 1)
    with pytest.raises(kp.InvalidArgument, match="out of range"):
        kp.mode_product(t, np.zeros((6, 9)), 7)
    with pytest.raises(kp.InvalidArgument, match="not square"):
        kp.KroneckerSum([np.zeros((2, 3))])
    with pytest.raises(kp.InvalidArgument, match="one factor per mode"):
        kp.tucker(t, [np.eye(3)])
    with pytest.raises(kp.InvalidArgument, match="n_steps"):
        kp.integrate_config("etd2rk", np.ones(3), [np.eye(3)], kp.G.zero(), 0.0, 1.0, 0)


def test_problem_builders_shapes_and_seeds(port):
    from paper_2304_02327_b200 import problems
    c = problems.ac2d(n=16)
    assert c.u0.shape == (16, 16) and c.u0.flags.f_contiguous and len(c.K) == 2
    assert np.array_equal(c.K[0], port.fd_operator_1d(16, 0.01))
    assert np.array_equal(problems.ac2d(n=16).u0, c.u0)  # seeded
    b = problems.brusselator(n=4)
    assert b.u0.shape == (4, 4, 4, 2) and b.K[3].shape == (2, 2) and not b.K[3].any()
    nl = problems.nls(n=8)
    assert nl.u0.dtype == np.complex128 and nl.K[0].dtype == np.complex128
    import pyoracle
    assert np.allclose(nl.K[0], 0.5j * pyoracle.periodic_laplacian_1d(8, 2.0))


def test_bench_reference_arm_contract():
    """bench.py --impl reference: one JSON line with the contract's keys, timed on
    the host cores (oracle/_ref when it is built, else the C restatement); under
    torchrun only rank 0 runs and prints."""
    import json
    import os
    import subprocess
    import sys
    from conftest import ROOT
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "1", "--n", "64"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["metric"].startswith("FP64 Tucker-op GFLOP/s") and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""
