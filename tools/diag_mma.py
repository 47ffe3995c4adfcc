"""MMA issue->commit and completion timing of CTA 0 / group 0 (diagnostic build)."""
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
print("records", n)
for k in range(4):
    r = rec[rec[:, 0] == k]
    if len(r):
        print("  kind", k, "issue cycles median", int(np.median(r[:, 2] - r[:, 1])), "count", len(r))
# last launch = bwd of block 0: its records are the last ones; wake times b[3800 + k*64 + it]
nt = sum(1 for x in rec[-200:] if x[0] == 3)  # G1' count in tail ~ ntiles of last launch
last = rec[-4 * nt - 1:] if nt else rec
for k in range(4):
    r = last[last[:, 0] == k]
    wake = b[3800 + k * 64: 3800 + k * 64 + len(r)]
    # G1 records include the prologue G1 of tile 0 (it=-1 -> tile 0)
    lat = [int(w - c) for w, c in zip(wake, r[:, 2]) if w > 0]
    print("  bwd kind", k, "commit->wake first tiles:", lat[:10], "median", int(np.median(lat)) if lat else None)
