"""The banded Kronecker-sum kernels (banded.cu): the defaults (v8 = v6 with the
z line in registers one plane ahead for complex tensors and species pairs, the
v6 lean line march for single real tensors), the v7 register-tiled march, the v2 march, the TMA
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


@pytest.mark.parametrize("variant", ["v2", "v3", "v4", "v5", "v6", "v7", "v8"])
def test_band_variant_bitwise(variant, default_hashes):
    assert probe({"KP_BAND": variant}) == default_hashes


@pytest.mark.parametrize("blocks", ["1", "16"])
def test_band_zchunk_bitwise(blocks, default_hashes):
    assert probe({"KP_BAND_BLOCKS": blocks}) == default_hashes


@pytest.mark.parametrize("env", [{"KP_BAND": "v7", "KP_B7_RY": "2"}, {"KP_BAND": "v7", "KP_B7_PF": "0"},
                                 {"KP_BAND": "v7", "KP_B7_BLOCKS": "1"},
                                 {"KP_BAND": "v7", "KP_B7_BLOCKS": "64"},
                                 {"KP_BAND": "v8", "KP_B8_MINB": "3"}, {"KP_BAND": "v8", "KP_B8_PF": "0"},
                                 {"KP_BAND": "v8", "KP_B8_BLOCKS": "1"}, {"KP_BAND": "v8", "KP_B8_HPF": "0"},
                                 {"KP_BAND": "v8", "KP_B8_YH": "1"}, {"KP_BAND": "v8", "KP_B8_MINB": "2"}])
def test_band78_shapes_bitwise(env, default_hashes):
    assert probe(env) == default_hashes
