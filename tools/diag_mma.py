"""Cycles the issuing warp spends in each tcgen05.mma chain (CTA 0, group 0),
by kernel and GEMM kind (diagnostic build with the REQ timing hook)."""
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
lib = _lib.load()
buf = torch.zeros(4096, dtype=torch.int64, device="cuda")
lib.fcg_debug_phase_buffer(_lib.vp(buf))
eng.evaluate()
torch.cuda.synchronize()
lib.fcg_debug_phase_buffer(None)
b = buf.cpu().numpy()
n = int(b[4095])
rec = b[1000:1000 + 3 * min(n, 900)].reshape(-1, 3)
names = {0: "G1", 1: "G2", 2: "G3", 3: "G1'"}
mmas = {(0, 0): 12, (0, 1): 24, (1, 0): 12, (1, 1): 24, (1, 2): 24, (1, 3): 12}
for kern in (0, 1):
    for k in range(4):
        r = rec[rec[:, 0] == k + 10 * kern]
        if len(r):
            med = int(np.median(r[:, 2] - r[:, 1]))
            print(("fwd", "bwd")[kern], names[k], "chain issue cycles median", med,
                  "per MMA", med // mmas[(kern, k)], "n", len(r))
