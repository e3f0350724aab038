"""The experiment harness (paper_2304_02327_b200/bench_runner.py, restating
src/bench_runner.cpp) and its CLI (tools/bench.cpp): host logic on CPU,
sweeps / selftest / CLI on the GPU."""
import io
import math

import numpy as np
import pytest

from paper_2304_02327_b200 import bench_runner as br


def test_observed_and_fit_order():
    errs = [1e-2, 2.5e-3, 6.25e-4]
    taus = [0.1, 0.05, 0.025]
    o = br.observed_order(errs, taus)
    assert o[0] == pytest.approx(2.0) and o[1] == pytest.approx(2.0)
    assert br.observed_order([1.0, 0.0], [0.1, 0.05]) == [None]
    assert br.fit_order(taus, errs) == pytest.approx(2.0)
    with pytest.raises(ValueError, match="two matched sweeps"):
        br.observed_order([1.0], [0.1])
    with pytest.raises(ValueError, match="two matched sweeps"):
        br.fit_order([0.1, 0.2], [1.0])


def test_default_steps():
    M = br.Method
    assert br.default_adr_steps(M.ETD2RK, 40) == [40, 140, 240, 340, 440]
    assert br.default_adr_steps(M.Lawson2b, 40)[-1] == 17500
    assert br.default_adr_steps(M.Lawson2b, 80)[-1] == 9000
    assert br.default_adr_steps(M.ExpEulerLinearSplit, 40) == [50, 450, 850, 1250, 1650]
    assert br.default_riccati_steps() == [30, 65, 100, 135, 170]
    with pytest.raises(ValueError):
        br.default_adr_steps(M.RosenbrockEuler, 40)


def test_csv_and_table_format(tmp_path):
    recs = [br.RunRecord("adr40", "etd2rk", 40, 0.025, 1.0 / 3.0, None, 0.5, 0.25),
            br.RunRecord("adr40", "etd2rk", 140, 1 / 140, 2e-5, 2.0123, 0.7, 0.5)]
    p = tmp_path / "r.csv"
    br.write_csv(str(p), recs)
    lines = p.read_text().splitlines()
    assert lines[0] == "problem,method,steps,tau,error,order,wallclock_s"
    assert lines[1] == "adr40,etd2rk,40,0.025000000000000001,0.33333333333333331,,0.5"
    assert lines[2].split(",")[5] == "2.0123000000000002"
    buf = io.StringIO()
    br.print_table(recs, buf)
    t = buf.getvalue().splitlines()
    assert t[0] == "adr40 / etd2rk"
    assert t[1] == "  " + "steps".ljust(12) + "40".rjust(12) + "140".rjust(12)
    assert t[3].split() == ["order", "--", "2.01"]


def test_cli_rejects_oracle_backend(capsys):
    from paper_2304_02327_b200 import cli
    with pytest.raises(SystemExit):
        cli.main(["adr", "--backend", "oracle"])


@pytest.mark.gpu
def test_run_adr_and_riccati_small(tmp_path, kp):
    out = io.StringIO()
    recs = br.run_adr(br.AdrOptions(10, 11, 12, ["etd2rk", "exp_euler"], [20, 40],
                                    str(tmp_path / "a.csv")), out)
    assert [r.n_steps for r in recs] == [20, 40, 20, 40]
    assert recs[1].observed_order == pytest.approx(2.0, abs=0.3)
    assert recs[3].observed_order == pytest.approx(1.0, abs=0.3)
    assert (tmp_path / "a.csv").read_text().count("\n") == 5
    rr = br.run_riccati(br.RiccatiOptions(6, [], [30, 60], 512, ""), out)
    assert [r.method for r in rr] == ["rosenbrock_euler"] * 2 + ["etd2rk"] * 2
    assert all(1.8 < r.observed_order < 2.2 for r in rr if r.observed_order is not None)


@pytest.mark.gpu
def test_run_steady_residual_decreases(kp, tmp_path):
    recs = br.run_steady(br.SteadyOptions(6, 40, 10, 0.2, ["etd2rk"], str(tmp_path / "s.csv")),
                         io.StringIO())
    res = [r.rel_residual for r in recs]
    assert len(res) == 4 and res[-1] < res[0]
    assert (tmp_path / "s.csv").read_text().startswith("problem,method,step,t,rel_residual\n")


@pytest.mark.gpu
def test_selftest_passes_and_catches_wrong_prefactor(kp):
    buf = io.StringIO()
    assert br.selftest(br.SelftestOptions(), buf), buf.getvalue()
    assert buf.getvalue().count("[PASS]") == 14
    bad = io.StringIO()
    assert not br.selftest(br.SelftestOptions(inject_wrong_prefactor=True), bad)
    assert "[FAIL] splitting error order (l=2" in bad.getvalue()


@pytest.mark.gpu
def test_cli_selftest_exit_code(kp, capsys):
    from paper_2304_02327_b200 import cli
    assert cli.main(["selftest"]) == 0
    assert "selftest: all checks passed" in capsys.readouterr().out
