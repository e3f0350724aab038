"""The banded Kronecker-sum kernels (banded.cu): the default v2 line march,
the TMA plane ring v3, the register z line v4 and v2 with its rows in shared
memory v5 (opt-in, KP_BAND) give
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


@pytest.mark.parametrize("variant", ["v3", "v4", "v5"])
def test_band_variant_bitwise(variant):
    assert probe({"KP_BAND": variant}) == probe({})
