"""Does the parity-split leaf form change how the error accumulates over steps?
Config 1, 60 steps: the runs with REXP_LEAF_DOWN_EO=0 / REXP_NO_LEAF_EO=1 against the default,
and all of them against the oracle golden at steps 1..3 (tests/golden/c1_steps.npz)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    from paper_1402_5168_b200 import api
    from workloads import CONFIGS
    g = np.load(os.path.join(ROOT, "tests/golden/c1_steps.npz"))
    cfg = CONFIGS[str(g["config"])]
    h = api.setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], cfg["Lambda_tau"] / cfg["tau"], f=cfg["f"])
    u = torch.from_numpy(np.ascontiguousarray(g["u0"][None])).to("cuda")
    out = []
    for s in range(1, 61):
        api.apply(h, u, 1)
        if s in (1, 2, 3, 5, 10, 20, 40, 60):
            torch.cuda.synchronize()
            out.append(u.cpu().numpy()[0].copy())
    np.save(sys.argv[2], np.stack(out))
    sys.exit(0)

runs = {"default": {}, "down_eo_off": {"REXP_LEAF_DOWN_EO": "0"}, "both_off": {"REXP_LEAF_DOWN_EO": "0", "REXP_NO_LEAF_EO": "1"}}
res = {}
for name, env in runs.items():
    path = f"/tmp/eo_{name}.npy"
    subprocess.check_call([sys.executable, __file__, "run", path], env={**os.environ, **env})
    res[name] = np.load(path)
g = np.load(os.path.join(ROOT, "tests/golden/c1_steps.npz"))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
steps = (1, 2, 3, 5, 10, 20, 40, 60)
for name in runs:
    print(name, "vs golden steps 1..3:", " ".join(f"{rel(res[name][i], g[f'u{i + 1}']):.2e}" for i in range(3)))
for name in ("down_eo_off", "both_off"):
    print("default vs", name, "at steps", steps, ":", " ".join(f"{rel(res['default'][i], res[name][i]):.2e}" for i in range(len(steps))))
print("down_eo_off vs both_off:", " ".join(f"{rel(res['down_eo_off'][i], res['both_off'][i]):.2e}" for i in range(len(steps))))
print("norms:", " ".join(f"{np.linalg.norm(res['default'][i]):.6e}" for i in range(len(steps))))
