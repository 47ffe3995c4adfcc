"""Diagnostic: dense large system, per-stage timing with syncs (GPU)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2602_13140_b200 import _lib
from paper_2602_13140_b200.engine import MDEngine
from paper_2602_13140_b200.inputs import generate_system
from paper_2602_13140_b200.modelparams import ModelConfig, init_params
kind, n, rc, bonded, R = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4] == "1", int(sys.argv[5])
sysm = generate_system(kind, n, 0, bonded=bonded)
params = init_params(ModelConfig(cutoff=rc), 0)
pos = np.repeat(sysm.positions[None], R, axis=0).astype(np.float32)
eng = MDEngine(params, sysm.types, sysm.masses, sysm.prior, R)
eng.load_state(pos, np.zeros_like(pos), 0)
print("cap", eng.cap_e, flush=True)
lib = _lib.load()
lib.fcg_profile_enable(1)
t = time.time(); eng.evaluate(); torch.cuda.synchronize(); print("evaluate s", time.time() - t, flush=True)
print(eng.flags(), "cap", eng.cap_e, flush=True)
print(_lib.profile_read(), flush=True)
lib.fcg_profile_enable(0)
