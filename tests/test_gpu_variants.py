"""Launch-configuration variants that are fixed once per process (read from the environment at
the first launch): each runs a cfg1 parity check in a fresh interpreter (-m gpu).

* MGNN_GATHER=reg      -- register gather (k_gather<false> for narrow rows, <true> for >= 128 floats)
* MGNN_GATHER=tma      -- TMA bulk copies (k_gather_g4 on these L2-resident tables; k_gather_tma with G4=0)
* MGNN_FLAT_BPS / MGNN_FLAT_UNR -- other block counts / loads in flight of the default k_gather_flat
* MGNN_PDL=0           -- plain launches instead of programmatic dependent launch
* MGNN_GATHER_HINT=0/3 -- (tma) no L2 cache hints / table rows evict_last and X rows evict_first
* MGNN_GATHER_HINT=10/14 (tma, G4=0) -- X rows stored through the LSU instead of bulk stores
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = """
import sys
sys.path.insert(0, {root!r})
from inputs import synth
from tests.parity_util import run_parity
g = synth.generate(synth.CONFIGS["cfg1"])
for D in (64, 200):
    run_parity(g, 2, D, [10, 25], 256, 2500, 0.9, 4, 1.0, [4, 4])
print("variant parity ok")
"""


@pytest.mark.parametrize("env", [{"MGNN_GATHER": "reg"}, {"MGNN_GATHER": "tma"},
                                 {"MGNN_GATHER": "tma", "MGNN_GATHER_G4": "0"},
                                 {"MGNN_FLAT_BPS": "3", "MGNN_FLAT_UNR": "8"}, {"MGNN_FLAT_UNR": "6"},
                                 {"MGNN_FLAT_BPS": "5", "MGNN_FLAT_UNR": "2"}, {"MGNN_PDL": "0"},
                                 {"MGNN_HOP_GRID_BPS": "0", "MGNN_COMPACT_BPS": "0"},
                                 {"MGNN_HOP_GRID_BPS": "5", "MGNN_COMPACT_BPS": "5"},
                                 {"MGNN_GATHER": "tma", "MGNN_GATHER_HINT": "0"},
                                 {"MGNN_GATHER": "tma", "MGNN_GATHER_HINT": "3"},
                                 {"MGNN_GATHER": "tma", "MGNN_GATHER_HINT": "10", "MGNN_GATHER_G4": "0"},
                                 {"MGNN_GATHER": "tma", "MGNN_GATHER_HINT": "14", "MGNN_GATHER_G4": "0"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_parity(env):
    """cfg1 parity under one environment variant (ids: the variables, e.g. MGNN_GATHER=flat)."""
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], cwd=ROOT, env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "variant parity ok" in r.stdout, (env, r.stdout[-2000:], r.stderr[-4000:])
