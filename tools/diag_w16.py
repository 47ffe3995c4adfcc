"""Per-atom energy differences of the W16 path against the golden oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import Golden
from helpers import params_for
from oracle import flashcg_oracle as O
import paper_2602_13140_b200 as P
g = Golden("flash")
for name in sys.argv[1:] or ["small_w16", "coil269_w16"]:
    c = g.case(name)
    params = params_for(c)
    out = P.flash_energy_forces(c["pos"], c["types"], params, P.PipelineMode())
    d = out.per_atom - c["per_atom"]
    print(name, os.environ.get("FCG_EDGE_IMPL", "tc"), "E err",
          O.energy_rel_err(out.energy, float(c["energy"]), c["per_atom"]),
          "F err", O.force_rel_err(out.forces, c["forces"]))
    idx = np.argsort(-np.abs(d))[:6]
    print("  worst atoms", [(int(i), float(d[i]), float(c["per_atom"][i])) for i in idx])
