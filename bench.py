#!/usr/bin/env python
"""Benchmark: repeated application of exp(tau L) ~ sum_m b_m (tau L - alpha_m)^{-1}
 on BASELINE.json's headline configuration.

A bench "step" = one big time step u <- R(tau L) u over the whole hot path
(all half poles, leaf solves, merge sweeps, pole sum, velocity recovery).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

N = 1: one process.  N > 1 (torchrun): the half poles are sharded across ranks
(pole-parallel "parallel in time"), each rank computes its
partial pole sums and an NCCL all-reduce sums them before the velocity
recovery ("scaling": "strong", the total work is one problem).
--impl reference times the CPU oracle (oracle/) on a bounded sample of poles.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, initial_state, wave_speed_field  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "dof-steps/s"
DEFAULT_CONFIG = "c3_rsw_32x32_p16_x64"   # the largest single-GPU BASELINE config


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_problem(cfg, x, y):
    kappa = wave_speed_field(x, y, cfg["seed"]) if cfg["model"] == "wave" else None
    return kappa


def tree_dims(n, q):
    """(nodes, n3, next) of every merge level (x-merge first, alternating), as in
    mesh.cpp: the x-merge reaching the full width closes the periodic x seam too
    (cylinder: n3 = both vertical seams, next = bottom + top)."""
    out = []
    ac = bc = 1
    lev = 0
    while True:
        if lev % 2 == 0:
            a, b = 2 * ac, bc
            if a == n:
                out.append((n // b, 2 * bc * q, 2 * n * q))
                return out
            n3 = bc * q
        else:
            a, b, n3 = ac, 2 * bc, ac * q
        out.append(((n // a) * (n // b), n3, 2 * (a + b) * q))
        ac, bc = a, b
        lev += 1


def class_work(cfg, nh, R2, shared, leaf="dense", nF=3, nE=3, sym2=False):
    """Algorithmic FP64 flops and operator bytes per step, per kernel class.
    Complex multiply-add = 8 flops, complex x real multiply-add = 4, complex
    product = 6; operator element = 16 bytes.  leaf = "spectral" counts the
    per-pole work of the spectral leaf kernels, per (half pole, leaf, real part);
    edge data live in the spectral edge basis, so neither kernel
    multiplies by V or V^-1 per pole:
      UP:   W = Dinv .* sum_f c_f G_f                          q^2 (4 nF + 6)
            y_s, z_s (4 weighted row/column sums) = the flux   16 q^2
      DOWN: boundary outer products b (4 complex x real)      16 q^2
            t = -c2 Dinv b, pole sums Re(d_k t)               q^2 (8 + 4 nE)
            owned edge segments' pole sums                    2q * 4 nE
    (the RHS-field part of the pole sum is pole-independent, sum_m Re(d_mk c_mf
    Dinv_m) =: Pi_kf, applied once per step in k_spec_back).  The once-per-step
    transforms (k_spec_pre_fused, k_spec_back) are O(q^3) per leaf, not per pole.
    """
    n, q = cfg["n"], cfg["p"] - 2
    q2, e = q * q, n * n
    lv = tree_dims(n, q)
    per = lambda nodes: 1 if shared else nodes
    # merge levels of the spectral shared store applied in symmetric-pair form
    # (device.cu: nodes * R2 <= 8 or R2 >= 16, not the first level): half the
    # operator bytes and flops
    sym = shared and leaf == "spectral"
    lv = [(nd, n3, nx, 0.5 if (sym and i > 0 and (nd * R2 <= 8 or R2 >= 16)) else 1.0)
          for i, (nd, n3, nx) in enumerate(lv)]
    # second reflection (device.cu: sym_pairs2, R2 >= 16): Y keeps half of the pair form's
    # rows and S half of its columns
    h2 = 0.5 if (sym2 and R2 >= 16) else 1.0
    y2 = lambda hf: hf * (h2 if hf < 1.0 else 1.0)
    merge = {
        "merge_up": (sum(nh * nd * (hf * n3 * n3 + y2(hf) * nx * n3) * R2 * 8 for nd, n3, nx, hf in lv),
                     sum(nh * per(nd) * (hf * n3 * n3 + y2(hf) * nx * n3) * 16 for nd, n3, nx, hf in lv)),
        # shared store: Fourier root (two DFTs over the n elements of the 2nq seam
        # unknowns, n blocks of (2q)^2); per-node: dense (2nq)^2
        "root": ((nh * R2 * (2 * 2 * n * q * n * 8 + n * (2 * q) ** 2 * 8), nh * n * (2 * q) ** 2 * 16) if shared
                 else (nh * (2 * n * q) ** 2 * R2 * 8, nh * (2 * n * q) ** 2 * 16)),
        "merge_down": (sum(y2(hf) * nh * nd * n3 * nx * R2 * 8 for nd, n3, nx, hf in lv),
                       sum(y2(hf) * nh * per(nd) * n3 * nx * 16 for nd, n3, nx, hf in lv)),
    }
    if leaf == "spectral":
        unit = nh * e * R2
        # the parity-split leaf GEMMs (leaf_gemm.cuh, round 2) execute fewer flops than the spectral FMA
        # form counted in round 1: UP 2q (o, r) x 2 rows x nF q x 2, DOWN 2q x (nE q + 2 nE) rows x 2 x 2
        # per (half pole, leaf, real RHS); the count is the smaller of the two (no credit for padding)
        up_fma, dn_fma = q2 * (4 * nF + 6 + 16), 16 * q2 + q2 * (8 + 4 * nE) + 8 * q * nE
        eo_up = os.environ.get("REXP_NO_LEAF_EO") is None
        mth = (nE * (q // 2) + nE + 7) // 8
        eo_dn = eo_up and q % 2 == 0 and 2 <= mth <= 4 and os.environ.get("REXP_LEAF_DOWN_EO") != "0"
        up_fl = min(up_fma, 8 * nF * q2) if eo_up else up_fma
        dn_fl = min(dn_fma, 8 * q * (nE * q + 2 * nE)) if eo_dn else dn_fma
        w = {
            "leaf_up": (unit * up_fl, nh * q2 * 16),
            "leaf_down": (unit * dn_fl, nh * q2 * 16),
        }
        w.update(merge)
        return w
    w = {
        "leaf_up": (nh * e * q2 * q2 * R2 * 8, nh * per(e) * q2 * q2 * 16),
        "leaf_flux": (nh * e * 4 * q * q * R2 * 4, 0),
        "leaf_down": (nh * e * q2 * 4 * q * R2 * 8, nh * per(e) * q2 * 4 * q * 16),
    }
    w.update(merge)
    return w


# FP64 peaks of this pool's B200 (MEASURED_PEAKS.json has no FP64 entry): measured
# with tools/fp64_peak.cu (profiles/r01_fp64_peak.txt); nominal 148 SMs x 64 FMA/clk
# x 2 x 1965 MHz = 37.2 TFLOP/s for both pipes.
FP64_DMMA_PEAK = 37.2
FP64_DFMA_PEAK = 35.93
PEAK_SOURCE = ("FP64: tools/fp64_peak.cu on this pool's B200 (profiles/r01_fp64_peak.txt): mma.sync.m8n8k4.f64 "
               "37.2, DFMA 35.93 TFLOP/s (= nominal 148 SM x 64 FMA x 2 x 1.965 GHz); HBM: MEASURED_PEAKS.json")


def class_bound(cls, shared, R2):
    """Which unit bounds a kernel class: the shared store's merge
    stages and leaf passes are DMMA GEMMs (k_cgemm / k_cgemm_sym / k_leaf_gemm_*; a
    few-RHS run's top levels are HBM-bound pair GEMVs), the Fourier root runs on
    the FP64 FMA pipe; the per-node store streams its operators (HBM)."""
    if not shared:
        return "hbm"
    if cls in ("merge_up", "merge_down", "leaf_up", "leaf_down"):
        return "tensor"   # the leaf passes are DMMA GEMMs over the poles (leaf_gemm.cuh) since round 2
    return "alu"


def state_bytes(cfg, nh, R2, shared, nF=3, nE=3):
    """Algorithmic bytes of the per-pole state each class must move per step
    (complex128 values x R2 real right-hand sides):
      merge up   X: read h^a_3, h^b_3 (2 n3), write w3 (n3); Y: read h_child[ext]
                 (next) and w3 (n3), write h (next)
      merge down read u_ext (next) and w3 (n3), write u3 (n3)
      root       read the 2 seam blocks of h (2 * 2nq), write s (2nq)
      leaf up    write the leaf flux (4q per leaf); read the RHS fields (nF q^2 reals) once per step
      leaf down  read the leaf's edge values (4q per leaf); write the pole sums (nE q^2 reals) once per step
    """
    n, q = cfg["n"], cfg["p"] - 2
    e = n * n
    lv = tree_dims(n, q)
    c = 16 * R2
    up = sum(nh * nd * (3 * n3 + 2 * nx + n3) * c for nd, n3, nx in lv)
    down = sum(nh * nd * (nx + 2 * n3) * c for nd, n3, nx in lv)
    root = nh * 3 * 2 * n * q * c
    leaf_up = nh * e * 4 * q * c + e * nF * q * q * 8 * R2
    leaf_down = nh * e * 4 * q * c + e * nE * q * q * 8 * R2
    return {"merge_up": up, "merge_down": down, "root": root, "leaf_up": leaf_up, "leaf_down": leaf_down}


def roofline_for(cfg, workload, h, times, steps, pk, step_ms, nh_here=None):
    """Dominant kernel = the class with the largest share of device time per
    step (CUDA events around every launch, on the launching stream).  achieved
    = algorithmic work per launch (class_work: flops, operator bytes; plus the
    per-pole state bytes of state_bytes) / average launch duration."""
    nh = nh_here or h.num_half_poles          # the half poles this handle applies
    R2 = 2 * h.nrhs
    shared = (cfg["model"] == "rsw")
    nF, nE = (3, 3) if cfg["model"] == "rsw" else (2, 2)
    work = class_work(cfg, nh, R2, shared, leaf=h.leaf_solver or "dense", nF=nF, nE=nE,
                      sym2="sym2[" in (h.stage_report or ""))
    sbytes = state_bytes(cfg, nh, R2, shared, nF, nE)
    hbm = pk.get("hbm_gbs", 6549.8)
    total_ms = sum(t for t, c in times.values())
    per_class = {}
    for k, (t, c) in times.items():
        if not c:
            continue
        d = {"share": round(t / total_ms, 4), "ms_per_step": round(t / steps, 4), "launches_per_step": c / steps}
        if k in work:
            fl, by = work[k]
            sb = sbytes.get(k, 0)
            sec = t / steps * 1e-3
            bound = class_bound(k, shared, R2)
            pkf = FP64_DMMA_PEAK if bound == "tensor" else FP64_DFMA_PEAK
            d.update({"bound": bound, "gflop_per_step": round(fl / 1e9, 3), "tflops": round(fl / sec / 1e12, 3),
                      "frac_fp64": round(fl / sec / 1e12 / pkf, 4),
                      "operator_GB_per_step": round(by / 1e9, 4), "state_GB_per_step": round(sb / 1e9, 4),
                      "GBps": round((by + sb) / sec / 1e9, 1), "frac_hbm": round((by + sb) / sec / 1e9 / hbm, 4)})
        per_class[k] = d
    dom = max((k for k in per_class if k in work), key=lambda k: times[k][0])
    ms, nl = times[dom]
    per_launch_ms = ms / max(nl, 1)
    lps = nl / steps
    fl, by = work[dom]
    bound = class_bound(dom, shared, R2)
    out = {"kernel": dom, "share_of_step": per_class[dom]["share"], "bound": bound,
           "per_launch_ms": round(per_launch_ms, 4), "launches_per_step": lps, "peak_source": PEAK_SOURCE,
           "traffic": traffic_for(workload, dom),
           "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/traffic.json)"}
    if bound == "hbm":
        ach = (by + sbytes.get(dom, 0)) / lps / (per_launch_ms * 1e-3) / 1e9
        out.update({"achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                    "algorithmic_bytes_per_launch": (by + sbytes.get(dom, 0)) / lps})
    else:
        pkf = FP64_DMMA_PEAK if bound == "tensor" else FP64_DFMA_PEAK
        ach = fl / lps / (per_launch_ms * 1e-3) / 1e12
        out.update({"achieved": round(ach, 3), "peak": pkf, "unit": "TFLOP/s", "frac": round(ach / pkf, 4),
                    "algorithmic_flops_per_launch": fl / lps})
    # whole step: every class's algorithmic work over the timed step time
    fl_all = sum(v[0] for v in work.values())
    by_all = sum(v[1] for v in work.values()) + sum(sbytes.values())
    out["whole_step"] = {"gflop": round(fl_all / 1e9, 2), "tflops": round(fl_all / (step_ms * 1e-3) / 1e12, 3),
                         "frac_fp64_tensor": round(fl_all / (step_ms * 1e-3) / 1e12 / FP64_DMMA_PEAK, 4),
                         "GB": round(by_all / 1e9, 3), "GBps": round(by_all / (step_ms * 1e-3) / 1e9, 1),
                         "frac_hbm": round(by_all / (step_ms * 1e-3) / 1e9 / hbm, 4)}
    out["per_class"] = per_class
    return out


def traffic_for(workload, kernel):
    """dram read+write bytes per launch of `kernel` in `workload`, from the committed
    ncu --set full capture (profiles/traffic.json, keyed "workload/class"), else None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d.get(f"{workload}/{kernel}")
    except Exception:
        return None


def oracle_sample(cfg, npoles_sample=None, nrhs_sample=2):
    """Time the CPU oracle on a bounded sample: `npoles_sample` of the poles
    (factorization untimed: it is the setup), one resolvent apply each per
    sampled RHS timed; the full-step time is extrapolated by the total pole
    count and the RHS count."""
    from oracle.models import RSW, Wave
    from oracle.rational import build_exp_approx
    from oracle.specelem import Mesh
    if npoles_sample is None:
        npoles_sample = 1 if cfg["n"] >= 32 else 2
    m = Mesh(cfg["n"], cfg["p"])
    model = RSW(m, cfg.get("f", 1.0)) if cfg["model"] == "rsw" else Wave(m, make_problem(cfg, m.x, m.y))
    ap = build_exp_approx(cfg["Lambda_tau"], cfg["delta"], verify=False)
    nr = min(nrhs_sample, cfg["nrhs"])
    U = [initial_state(cfg["model"], m.x, m.y, cfg["seed"] + 10 * k) for k in range(nr)]
    P = len(ap["poles"])
    idx = np.linspace(0, P - 1, npoles_sample + 2).astype(int)[1:-1]
    solve_s = 0.0
    factor_s = 0.0
    for k in idx:
        t0 = time.perf_counter()
        lu = model.factor(ap["poles"][k] / cfg["tau"])
        factor_s += time.perf_counter() - t0
        t0 = time.perf_counter()
        for u0 in U:
            _ = ap["res"][k] * model.resolvent(ap["poles"][k], cfg["tau"], u0, lu=lu)
        solve_s += time.perf_counter() - t0
        del lu
    step_s = solve_s / (len(idx) * nr) * P * cfg["nrhs"]
    dof = 3 * m.N * cfg["nrhs"]
    return {"value": dof / step_s, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{len(idx)} of {P} poles x {nr} of {cfg['nrhs']} RHS on the full "
                      f"{cfg['n']}x{cfg['n']}x{cfg['p']}^2 mesh, one resolvent apply each (scipy splu + two "
                      f"refinement steps, single-threaded; factor untimed, {factor_s:.1f}s), step time extrapolated "
                      f"x{P}/{len(idx)} poles x{cfg['nrhs']}/{nr} RHS",
            "step_seconds": step_s}


def bench_config(workload, cfg, poles, N):
    """The `config` object of both arms (identical keys and values)."""
    return {"workload": workload, "model": cfg["model"], "elements": f"{cfg['n']}x{cfg['n']}", "p": cfg["p"],
            "Lambda_tau": cfg["Lambda_tau"], "tau": cfg["tau"], "delta": cfg["delta"], "nrhs": cfg["nrhs"],
            "poles": poles, "dof": 3 * N * cfg["nrhs"], "nodes_per_field": N,
            "baseline_nodes_per_field_convention": cfg["n"] ** 2 * cfg["p"] ** 2,
            "l2": "operator store + work buffers exceed the 126 MB L2 (no flush needed)"}


# The paper's own comparison (context, not the target): PAPER.md Tables 2 and 3
# (PAPER.md:903-928, 1068-1089), all methods in Octave, hardware
# not stated; 12 x 12 elements of 16 x 16 nodes, one application of e^{1.5 L}.
PAPER_CONTEXT = {
    "source": "PAPER.md Table 2 (RSW, PAPER.md:903-928) and Table 3 (wave, PAPER.md:1068-1089); Octave "
              "implementations (PAPER.md:966-967); hardware not stated",
    "setup": "12x12 elements, 16x16 Chebyshev nodes each, one apply of exp(1.5 L), M = 376 terms",
    "rsw_minutes": {"rational_apply": 4.39, "rational_precompute": 103.1, "rk4": 131.9, "chebyshev_deg12": 150.5},
    "wave_minutes": {"rational_apply": 3.76, "rational_precompute": 113.4, "rk4": 63.9, "chebyshev_deg12": 57.5},
    "rsw_rational_dof_steps_per_s": round(3 * 144 * 224 / (4.39 * 60), 1),
}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.rational import build_exp_approx
    from oracle.specelem import Mesh
    t0 = time.perf_counter()
    res = oracle_sample(cfg)
    poles = len(build_exp_approx(cfg["Lambda_tau"], cfg["delta"], verify=False)["poles"])
    N = Mesh(cfg["n"], cfg["p"]).N
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["step_seconds"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic", "config": bench_config(args.config, cfg, poles, N),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "paper_context": PAPER_CONTEXT, "wall_s": round(time.perf_counter() - t0, 1)}
    print(json.dumps(line), flush=True)


def pernode_bytes_per_half_pole(cfg):
    """Per-node store bytes of one half pole: dense leaf A_II^-1
    (q^2 x q^2) and S_leaf (q^2 x 4q) per element, X / Y / S per merge-tree
    node, dense periodic root (2nq)^2 - complex128."""
    n, q = cfg["n"], cfg["p"] - 2
    q2 = q * q
    leaf = n * n * (q2 * q2 + q2 * 4 * q)
    levs = sum(nd * (n3 * n3 + 2 * n3 * nx) for nd, n3, nx in tree_dims(n, q))
    return 16 * (leaf + levs + (2 * n * q) ** 2)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1402_5168_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    Lam = cfg["Lambda_tau"] / cfg["tau"]

    # setup (untimed): poles, factorization, device store
    t_setup = time.perf_counter()
    kappa = None
    if cfg["model"] == "wave":
        xm, ym = api.mesh_coords(cfg["n"], cfg["p"])
        kappa = wave_speed_field(xm, ym, cfg["seed"])
    common = dict(f=cfg.get("f", 1.0), kappa=kappa, nrhs=cfg["nrhs"])
    nh_total = None
    if world > 1 or args.shard is not None:
        tmp = api.setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, device=-1,
                        half_range=(0, 1), **common)
        nh_total = tmp.num_half_poles
        tmp.close()
    shard = None
    if args.shard is not None:
        # one rank's share of a pole-sharded run on this GPU: the largest number of
        # half poles whose per-node store fits (or the requested count)
        if world > 1:
            raise SystemExit("--shard is a single-GPU measurement")
        per = pernode_bytes_per_half_pole(cfg)
        free, total = torch.cuda.mem_get_info(dev)
        fit = int((free - 24 * 2 ** 30) // per)
        k = fit if args.shard == "auto" else min(int(args.shard), fit)
        k = max(1, min(k, nh_total))
        shard = (0, k)
        h = api.setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, device=local,
                      half_range=shard, **common)
    elif world > 1:
        from paper_1402_5168_b200.parallel import half_range
        lo, hi = half_range(nh_total, rank, world)
        h = api.setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, device=local,
                      half_range=(lo, hi), **common)
    else:
        h = api.setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, device=local, **common)
        nh_total = h.num_half_poles
    t_setup = time.perf_counter() - t_setup
    x, y = h.node_coords()
    N = h.N
    u0 = np.stack([initial_state(cfg["model"], x, y, cfg["seed"] + 10 * k) for k in range(cfg["nrhs"])])
    u = torch.from_numpy(u0).to(dev).contiguous()
    stream = torch.cuda.current_stream(dev)
    sharded = world > 1 or shard is not None
    e = torch.zeros(h.partial_len, dtype=torch.float64, device=dev) if sharded else None

    def one_step():
        if not sharded:
            api.apply(h, u, 1)
        else:
            api.step_partial(h, u, e)
            if world > 1:
                dist.all_reduce(e)
            api.step_finish(h, e, u)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # the production path (one CUDA graph per step); cudaProfilerStart/Stop
        # bracket the timed steps, so `ncu --profile-from-start off ... bench.py`
        # lists exactly these launches
        torch.cuda.profiler.start()
        ev0.record(stream)
        for _ in range(args.steps):
            one_step()
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.profiler.stop()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    # per-kernel breakdown in a separate pass (events around every launch on the
    # launching stream; eager launches), not part of the timed value
    api.timing_begin(h)
    for _ in range(args.steps):
        one_step()
    torch.cuda.synchronize()
    kt = api.timing_end(h)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    dof = 3 * N * cfg["nrhs"]
    value = dof * args.steps / (ms * 1e-3)
    finite = bool(torch.isfinite(torch.view_as_real(u)).all().item())

    # end-to-end through the public C ABI with HOST buffers: every step copies the
    # state in from pinned host memory, steps, and reads it back (rexp_apply host path)
    e2e = None
    if world == 1 and shard is None:
        uh = torch.from_numpy(u0.copy()).pin_memory()
        uh_np = uh.numpy()
        for _ in range(max(1, args.warmup)):
            api.apply(h, uh_np, 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            api.apply(h, uh_np, 1)
        te = time.perf_counter() - t0
        sb = u0.nbytes
        e2e = {"value": dof * args.steps / te, "unit": UNIT, "h2d_bytes_per_step": sb, "d2h_bytes_per_step": sb,
               "timing": "host wall clock around K synchronous rexp_apply(host ptr, 1 step) calls"}

    pk = peaks()
    nh_here = (shard[1] - shard[0]) if shard else (hi - lo) if world > 1 else nh_total
    roof = roofline_for(cfg, args.config, h, kt, args.steps, pk, ms / args.steps, nh_here)
    launches = sum(v[1] for v in kt.values())
    conf = bench_config(args.config, cfg, h.num_poles, N)
    conf["parallelism"] = (f"pole-sharded x{world}" if world > 1 else
                           (f"one shard of a pole-sharded run: half poles [{shard[0]}, {shard[1]}) of {nh_total}"
                            if shard else "single GPU"))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64)", "data": "synthetic",
            "config": conf,
            "impl_details": {"half_poles_total": nh_total, "half_poles_here": h.num_half_poles if shard is None
                             else shard[1] - shard[0],
                             "store": "shared" if cfg["model"] == "rsw" else "pernode",
                             "leaf_solver": h.leaf_solver, "merge_kernels": h.stage_report,
                             "store_bytes": h.store_bytes, "work_bytes": h.work_bytes},
            "roofline": roof,
            "kernel_ms": {k: round(v[0], 3) for k, v in kt.items()},
            "gpu_launches": launches, "e2e": e2e,
            "clocks": clk.summary(), "setup_s": round(t_setup, 1), "finite": finite,
            "paper_context": PAPER_CONTEXT}
    if shard is not None:
        per = pernode_bytes_per_half_pole(cfg)
        line["shard"] = {
            "half_poles": shard[1] - shard[0], "half_poles_total": nh_total,
            "store_bytes_per_half_pole": per, "store_bytes_measured": h.store_bytes,
            "full_store_bytes": per * nh_total,
            "gpus_needed_for_full_store": math.ceil(per * nh_total / (torch.cuda.mem_get_info(dev)[1] - 24 * 2 ** 30)),
            "value_meaning": "dof-steps/s of this shard's step (its half poles' pole sums + recovery); the full "
                             "job on one GPU would run at value x half_poles / half_poles_total if it fit",
            "full_job_equivalent": value * (shard[1] - shard[0]) / nh_total}
    if rank == 0:
        if world == 1 and shard is None and not args.no_cpu_baseline:
            try:
                cb = oracle_sample(cfg)
                line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            except Exception as ex:  # pragma: no cover
                line["cpu_baseline"] = {"error": str(ex)}
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default=None,
                    help="'auto' or a half-pole count: time one rank's shard of a pole-sharded run on this GPU "
                         "(configs whose store does not fit one B200: c2, c4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
