"""Golden traffic reports of every PipelineMode schedule, made by running
the REFERENCE (flashcg) here:
    python tests/golden/make_traffic_golden.py
-> tests/golden/traffic_modes.json (committed).  Pins the modelled-traffic
bookkeeping of the ablation schedules (flash.py:310-443, traffic.py:80-182)
that paper_2602_13140_b200.schnet.traffic_report restates.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from flashcg import flash as RF  # noqa: E402
from flashcg import model as RM  # noqa: E402
from flashcg import systems as RS  # noqa: E402


def main():
    cases = []
    for kind, n, seed, cfg in (("coil", 40, 0, dict(hidden_dim=16, rbf_dim=8, num_blocks=2,
                                                       cutoff=1.0, num_atom_types=8,
                                                       filter_hidden_dim=16,
                                                       readout_hidden_dim=8)),
                               ("globule", 30, 1, {})):
        sysm = RS.generate_system(kind, n, seed)
        params = RM.init_params(RM.ModelConfig(**cfg), 3)
        for dtype in (np.float32, np.float64):
            p = params if dtype == np.float32 else params.astype(np.float64)
            pos = sysm.positions.astype(dtype)
            for fused in (True, False):
                for segred in (True, False):
                    mode = RF.PipelineMode(fused=fused, segred=segred)
                    out = RF.flash_energy_forces(pos, sysm.types, p, mode)
                    cases.append(dict(kind=kind, n=n, seed=seed, pseed=3, cfg=cfg,
                                      dtype=np.dtype(dtype).name, fused=fused, segred=segred,
                                      traffic=out.traffic.as_dict()))
    (OUT / "traffic_modes.json").write_text(json.dumps(cases, indent=1, sort_keys=True) + "\n")
    print(f"{len(cases)} traffic reports")


if __name__ == "__main__":
    main()
