"""Energy/force relative errors against the oracle for one configuration,
for whichever edge implementation the environment selects (diagnostic).

    FCG_EDGE_IMPL=simt python tools/diag_precision.py globule 2000 2.0
"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import flashcg_oracle as O
from paper_2602_13140_b200.engine import MDEngine
from paper_2602_13140_b200.inputs import generate_system
from paper_2602_13140_b200.modelparams import ModelConfig, init_params

kind, n, rc = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
sysm = generate_system(kind, n, 0, bonded=(kind != "globule"))
params = init_params(ModelConfig(cutoff=rc), 0)
R = 2
rng = np.random.default_rng(n)
pos = (sysm.positions[None] + rng.normal(0, 0.01, size=(R, n, 3))).astype(np.float32)
eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R)
eng.load_state(pos, np.zeros_like(pos), 0)
eng.evaluate()
Fm = eng.model_forces.cpu().numpy()
pot = eng.potential.cpu().numpy()
pa = eng.per_atom.cpu().numpy().reshape(R, n)
for r in range(R):
    e, pa_ref, f = O.energy_forces(pos[r], sysm.types, params)
    # the oracle's own fp64 evaluation of the same fp32 inputs
    e64, pa64, f64 = O.energy_forces(pos[r].astype(np.float64), sysm.types, params.astype(np.float64))
    print(f"replica {r}: gpu-vs-oracle32 E {O.energy_rel_err(float(pot[r]), e, pa_ref):.2e} "
          f"F {O.force_rel_err(Fm[r], f):.2e} | gpu-vs-oracle64 E {O.energy_rel_err(float(pot[r]), e64, pa64):.2e} "
          f"F {O.force_rel_err(Fm[r], f64):.2e} | oracle32-vs-64 E {O.energy_rel_err(e, e64, pa64):.2e} "
          f"F {O.force_rel_err(f, f64):.2e} | per-atom max rel {np.max(np.abs(pa[r]-pa_ref))/np.max(np.abs(pa_ref)):.2e}")
