"""The banded Kronecker-sum kernels (banded.cu): the default v6 lean line
march (real tensors; v2 for complex / species pairs), the v2 march, the TMA
plane ring v3, the register z line v4, v2 with its rows in shared memory v5
and v6 for every form (opt-in, KP_BAND), and other z-chunk lengths
(KP_BAND_BLOCKS) give
BIT-IDENTICAL Kronecker sums and integrations (same values into the same row
chains).  One process per variant (the switch is read once)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def probe(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "band_probe.py")], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.split()


@pytest.fixture(scope="module")
def default_hashes():
    return probe({})


@pytest.mark.parametrize("variant", ["v2", "v3", "v4", "v5", "v6"])
def test_band_variant_bitwise(variant, default_hashes):
    assert probe({"KP_BAND": variant}) == default_hashes


@pytest.mark.parametrize("blocks", ["1", "16"])
def test_band_zchunk_bitwise(blocks, default_hashes):
    assert probe({"KP_BAND_BLOCKS": blocks}) == default_hashes
