"""Every kernel variant reachable through an environment knob (A/B switches,
defaults = measured best) stays bit-identical to the CPU oracle."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

KNOBS = [
    {},
    {"BOYS_PDL": "0"},
    {"BOYS_SOA_PAIR": "0"},
    {"BOYS_SOA_PAIR": "0", "BOYS_GRID_TILES": "1"},
    {"BOYS_GRID_TILES": "2", "BOYS_PAIR_GRID": "2"},
    {"BOYS_PAIR_GRID": "1"},
    {"BOYS_SOA_TMA": "1", "BOYS_SOA_PAIR": "0"},
    {"BOYS_AOS_NBUF": "1"},
    {"BOYS_AOS_PAIR": "1"},
    {"BOYS_AOS_PAIR": "0"},
    {"BOYS_SOA_QUAD": "1"},
    {"BOYS_SOA_QUAD": "0"},
    {"BOYS_AOS_VEC": "1"},
    {"BOYS_AOS_VEC": "0"},
    {"BOYS_AOS_NBUF": "1", "BOYS_AOS_MINB": "6"},
    {"BOYS_SOA0_MINB": "6", "BOYS_SOA_PAIR": "0"},
    {"BOYS_RAGGED_EPL": "1"},
    {"BOYS_RAGGED_GRID_MULT": "3"},
]


@pytest.mark.parametrize("env", KNOBS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "defaults")
def test_knob_parity(env):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "knob_parity.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
