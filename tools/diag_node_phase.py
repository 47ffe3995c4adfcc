"""Per-phase timing of the node kernels (needs a -DFCG_NODE_STAMPS build,
e.g. FCG_LIB_PATH=.../libfcg_b.so).  Kinds: 0 pre, 1 pre_bwd, 2 post,
3 post_bwd, 4 readout; the last launch of each kind is recorded."""
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
buf = torch.zeros(4096 + 5 * 1024 * 8, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.fcg_debug_phase_buffer(_lib.vp(buf))
for _ in range(3):
    eng.evaluate()
torch.cuda.synchronize()
lib.fcg_debug_phase_buffer(None)
eng.evaluate()
b = buf[4096:].cpu().numpy().reshape(5, 1024, 8)
names = {0: ("pre", [1, 2, 3, 4]), 1: ("pre_bwd", [1, 2, 3, 4]), 2: ("post", [1, 2, 3, 4, 5]),
         3: ("post_bwd", [1, 2, 3, 5]), 4: ("readout", [1, 2, 3, 5])}
if os.environ.get("FCG_NODE_FUSE", "1") != "0":  # k_node_post_pre_tc: post part (kind 2), pre part (kind 0)
    names = {2: ("post_pre:post", [1, 2, 3, 4, 5]), 0: ("post_pre:pre", [1, 2, 3])}
for k, (name, phs) in names.items():
    t = b[k]
    ok = t[:, 6] > 0
    t = t[ok]
    if not len(t):
        continue
    span_ns = t[:, 7].max() - t[:, 6].min()
    cta_ns = np.median(t[:, 7] - t[:, 6])
    start_spread = np.percentile(t[:, 6] - t[:, 6].min(), [50, 90, 100])
    d = [np.median(t[:, p] - t[:, q]) for q, p in zip([0] + phs[:-1], phs)]
    print(f"{name:9s} ctas {ok.sum():4d} span {span_ns/1e3:6.2f} us  cta median {cta_ns/1e3:5.2f} us  "
          f"start spread p50/p90/max {start_spread/1e3} us")
    print("   phase cycles (prologue, ...):", [int(x) for x in d])
