"""The selectable alternative kernels keep parity.

The library reads its kernel switches once per process, so each setting runs
the fp32 / W16 energy-force parity tests and the batched-engine test of
test_gpu_parity.py in a subprocess (settings: space-separated VAR=value):

  * FCG_FWD_WS=0: the 64-edge forward with last-arriver MMA issue
    (k_edge_fwd64); with FCG_FWD64=0 the 4-group, 32-edge forward;
  * FCG_BWD_WS=0: the forward-mode backward with last-arriver issue
    (k_edge_bwd_fm); FCG_BWD_UPG=1 its 4 x 4-warp shape; FCG_BWD_FM=0 the
    reverse-mode 64-edge backward (k_edge_bwd64); with FCG_BWD64=0 too the
    4-group, 32-edge one (k_edge_bwd_tc);
  * FCG_EDGE_IMPL=simt: the SIMT edge kernels (with the separate k_embed);
  * FCG_NODE_FUSE=0: one launch per node stage instead of the fused
    post+pre, post+readout+post_bwd and pre_bwd+post_bwd launches;
  * FCG_NBR_FUSED=0 / FCG_NBR_WINDOW=0: the general neighbour builds, run
    through the CSR and large-system tests instead.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _run(setting, sel):
    env = dict(os.environ, **dict(kv.split("=") for kv in setting.split()))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu",
                        "-q", "-x", "-p", "no:cacheprovider", "-k", sel],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "deselected" in r.stdout


@pytest.mark.parametrize("setting", ["FCG_FWD_WS=0", "FCG_FWD_WS=0 FCG_FWD64=0", "FCG_BWD_WS=0",
                                     "FCG_BWD_WS=0 FCG_BWD_UPG=1", "FCG_BWD_FM=0",
                                     "FCG_BWD_FM=0 FCG_BWD64=0", "FCG_EDGE_IMPL=simt",
                                     "FCG_NODE_FUSE=0"])
def test_alternative_edge_kernels_match_oracle(setting):
    _run(setting, "energy_forces_fp32 or energy_forces_w16 or batched_engine_matches_oracle")


@pytest.mark.parametrize("setting", ["FCG_NBR_FUSED=0", "FCG_NBR_WINDOW=0"])
def test_alternative_neighbour_builds_match_oracle(setting):
    _run(setting, "csr or large_system_sweep or neighbor")
