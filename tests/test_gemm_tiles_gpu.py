"""Every tile configuration of the GEMM (gemm_dmma.cu menu, forced with
KP_GEMM_TILE; B = the balanced 112-row / 112-column tiles incl. the stacked
"flat" row blocks of batched products, KP_GEMM_BAL=2 single-wave products / 1 also multi-wave) and the cp.async producer (KP_TMA=0) give BIT-IDENTICAL mode
products, Tucker operators and complex products: the k order of every
accumulator is the same in all of them (DMMA k-slot t of k-step s holds
k = 16 kt + 4 s + t, in order).  Each variant runs in its own process (the
switches are read once)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def probe(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tile_probe.py")], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.split()


@pytest.fixture(scope="module")
def default_hashes():
    return probe({})


@pytest.mark.parametrize("variant", [{"KP_GEMM_TILE": t} for t in "SMNLGB"] +
                         [{"KP_TMA": "0"}, {"KP_TMA": "0", "KP_GEMM_TILE": "G"},
                          {"KP_GEMM_BAL": "2"}, {"KP_GEMM_BAL": "1"}, {"KP_FUSE01": "0"}])
def test_tile_variant_bitwise(default_hashes, variant):
    assert probe(variant) == default_hashes
