"""Timeline of the 64-edge forward and the forward-mode backward edge
kernels (CTA 0, first warp of each group) from a -DFCG_EDGE_STAMPS build:
median cycles per phase over iterations 2..29.

    FCG_NVCC_EXTRA=-DFCG_EDGE_STAMPS build -> libfcg_b.so, then
    FCG_LIB_PATH=.../libfcg_b.so python tools/diag_edge_timeline.py
"""
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
buf = torch.zeros(2 * 2 * 32 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.fcg_debug_phase_buffer(_lib.vp(buf))
eng.evaluate()
torch.cuda.synchronize()
lib.fcg_debug_phase_buffer(None)
b = buf.cpu().numpy().reshape(2, 2, 32, 16).astype(np.int64)
names = {0: ("fwd64", ["wait G1", "E1 h", "ready G2", "basis+ready G1", "wait G2", "E2", "gathers"]),
         1: ("bwd_fm", ["wait G1", "E1 h,v", "ready G2|G3", "gathers+basis", "wait G2|G3", "E2 seg+u", "q+G1+red", "xg exchange"])}
for k, (nm, ph) in names.items():
    for g in range(2):
        t = b[k, g]
        ok = t[:, 0] > 0
        its = np.nonzero(ok)[0]
        its = its[(its >= 2) & (its < 30)]
        if len(its) < 3:
            continue
        n = len(ph) + 1
        d = np.array([np.diff(t[i, :n]) for i in its])
        per = np.array([t[i + 1, 0] - t[i, 0] for i in its if i + 1 < 32 and t[i + 1, 0] > 0])
        print(f"{nm} group {g}: iteration {int(np.median(per))} cycles; " +
              ", ".join(f"{p} {int(np.median(d[:, j]))}" for j, p in enumerate(ph)))
