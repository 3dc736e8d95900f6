"""Profile exactly one warm step of a workload (for ncu --profile-from-start off).

    ncu --profile-from-start off --set full --clock-control none \
        python tools/profile_step.py --config c1_rsw_16x16_p16

Setup (factorization, upload, autotuning) and two warm-up steps run outside
the profiled range; cudaProfilerStart/Stop bracket one step.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1402_5168_b200 import api  # noqa: E402
from workloads import CONFIGS, initial_state, wave_speed_field  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1_rsw_16x16_p16", choices=sorted(CONFIGS))
    ap.add_argument("--warm", type=int, default=2)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    n, p = cfg["n"], cfg["p"]
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    x, y = api.mesh_coords(n, p)
    kappa = wave_speed_field(x, y, cfg["seed"]) if cfg["model"] == "wave" else None
    h = api.setup(cfg["model"], n, p, cfg["tau"], cfg["delta"], Lam, f=cfg.get("f", 1.0), kappa=kappa,
                  nrhs=cfg["nrhs"])
    u0 = np.stack([initial_state(cfg["model"], x, y, cfg["seed"] + 10000 * r) for r in range(cfg["nrhs"])])
    u = torch.from_numpy(u0).to("cuda")
    api.apply(h, u, args.warm)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    api.apply(h, u, 1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step of", args.config, "finite:", bool(torch.isfinite(torch.view_as_real(u)).all()))


if __name__ == "__main__":
    main()
