"""Accuracy experiment: one c1 step against the oracle golden (tests/golden/c1_steps.npz),
with the error split by field and by node class.  Usage: python tools/c1_err.py [tag]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1402_5168_b200 import api  # noqa: E402
from workloads import CONFIGS  # noqa: E402

g = np.load(os.path.join(ROOT, "tests/golden/c1_steps.npz"))
cfg = CONFIGS[str(g["config"])]
h = api.setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], cfg["Lambda_tau"] / cfg["tau"], f=cfg["f"], nrhs=1)
u = torch.from_numpy(np.ascontiguousarray(g["u0"][None])).to("cuda")
out = []
for s in (1, 2, 3):
    api.apply(h, u, 1)
    torch.cuda.synchronize()
    got = u.cpu().numpy()[0]
    ref = g[f"u{s}"]
    e = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    per = [np.linalg.norm(got[f] - ref[f]) / np.linalg.norm(ref) for f in range(3)]
    out.append(f"step{s} {e:.3e} fields " + " ".join(f"{x:.2e}" for x in per))
    if s == 1:
        d = np.abs(got - ref).max(axis=0)
        NI = cfg["n"] ** 2 * (cfg["p"] - 2) ** 2
        out.append(f"  max|err| interior {d[:NI].max():.2e} edges {d[NI:].max():.2e} |ref|max {np.abs(ref).max():.2e}")
print(sys.argv[1] if len(sys.argv) > 1 else "", "|", h.stage_report)
print("\n".join(out), flush=True)
