"""Per-phase cycle breakdown of the tcgen05 edge kernels (CTA 0, group 0)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_13140_b200 import _lib
from paper_2602_13140_b200.engine import MDEngine
from paper_2602_13140_b200.inputs import generate_system
from paper_2602_13140_b200.modelparams import ModelConfig, init_params
sysm = generate_system("coil", 269, 0)
params = init_params(ModelConfig(), 0)
R = 64
pos = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R)
eng.load_state(pos, np.zeros_like(pos), 0)
eng.evaluate()
buf = torch.zeros(2 * 16 * 64, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.fcg_debug_phase_buffer(_lib.vp(buf))
eng.evaluate()
torch.cuda.synchronize()
lib.fcg_debug_phase_buffer(None)
b = buf.cpu().numpy().reshape(2, 16, 64)
for kind, name, nph in ((0, "fwd", 6), (1, "bwd", 11)):
    t = b[kind, :, :nph].astype(np.int64)
    ok = t[:, 0] > 0
    t = t[ok]
    d = np.diff(t, axis=1)
    tile = t[1:, 0] - t[:-1, 0]
    print(name, "tiles", ok.sum(), "cycles/tile", np.median(tile) if tile.size else None)
    print("  phase medians:", [int(x) for x in np.median(d, axis=0)])
