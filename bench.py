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
DEFAULT_CONFIG = "c1_rsw_16x16_p16"


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


def class_work(cfg, nh, R2, shared, leaf="dense", nF=3, nE=3):
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
    merge = {
        "merge_up": (sum(hf * nh * nd * (n3 * n3 + nx * n3) * R2 * 8 for nd, n3, nx, hf in lv),
                     sum(hf * nh * per(nd) * (n3 * n3 + nx * n3) * 16 for nd, n3, nx, hf in lv)),
        # shared store: Fourier root (two DFTs over the n elements of the 2nq seam
        # unknowns, n blocks of (2q)^2); per-node: dense (2nq)^2
        "root": ((nh * R2 * (2 * 2 * n * q * n * 8 + n * (2 * q) ** 2 * 8), nh * n * (2 * q) ** 2 * 16) if shared
                 else (nh * (2 * n * q) ** 2 * R2 * 8, nh * (2 * n * q) ** 2 * 16)),
        "merge_down": (sum(hf * nh * nd * n3 * nx * R2 * 8 for nd, n3, nx, hf in lv),
                       sum(hf * nh * per(nd) * n3 * nx * 16 for nd, n3, nx, hf in lv)),
    }
    if leaf == "spectral":
        unit = nh * e * R2
        w = {
            "leaf_up": (unit * q2 * (4 * nF + 6 + 16), nh * q2 * 16),
            "leaf_down": (unit * (16 * q2 + q2 * (8 + 4 * nE) + 8 * q * nE), nh * q2 * 16),
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


def roofline_for(cfg, h, times, steps, pk):
    """Dominant kernel = the class with the largest device time.  achieved =
    algorithmic work per launch / average launch time (CUDA events on the
    launching stream)."""
    nh = h.num_half_poles
    R2 = 2 * h.nrhs
    shared = (cfg["model"] == "rsw")
    nF, nE = (3, 3) if cfg["model"] == "rsw" else (2, 2)
    work = class_work(cfg, nh, R2, shared, leaf=h.leaf_solver or "dense", nF=nF, nE=nE)
    # dominant kernel = the single launch with the largest average duration
    # (the merge tree is many launches of different shapes; it is reported per class)
    # (among the classes with a work model: the per-step pre/recover/pole-sum
    # kernels are small and bandwidth-trivial)
    dom = max((k for k in times if times[k][1] and k in work), key=lambda k: times[k][0] / times[k][1])
    ms, nl = times[dom]
    per_launch_ms = ms / max(nl, 1)
    # the spectral leaf kernels run on the FP64 FMA pipe: measured DFMA 35.9 TFLOP/s
    # (profiles/r01_fp64_peak.txt; nominal 148 SMs x 64 FMA/clk x 2 x 1965 MHz = 37.2)
    fp64_peak = 35.93
    per_class = {}
    for k, (t, c) in times.items():
        if k in work and c:
            fl, by = work[k]
            launches_per_step = c / steps
            sec = t / c * 1e-3
            per_class[k] = {"tflops": round(fl / launches_per_step / sec / 1e12, 3),
                            "operator_GBps": round(by / launches_per_step / sec / 1e9, 1)}
    if dom not in work:
        return {"kernel": dom, "bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None, "per_class": per_class}
    fl, by = work[dom]
    lps = nl / steps
    if shared:
        ach = fl / lps / (per_launch_ms * 1e-3) / 1e12
        return {"kernel": dom, "bound": "alu", "achieved": round(ach, 3), "peak": round(fp64_peak, 2),
                "unit": "TFLOP/s", "frac": round(ach / fp64_peak, 4), "traffic": traffic_for(dom),
                "peak_source": "measured DFMA 35.93 TF (profiles/r01_fp64_peak.txt, tools/fp64_peak.cu); nominal 37.2",
                "per_launch_ms": round(per_launch_ms, 4), "per_class": per_class}
    hbm = pk.get("hbm_gbs", 6650.0)
    ach = by / lps / (per_launch_ms * 1e-3) / 1e9
    return {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": traffic_for(dom), "peak_source": "MEASURED_PEAKS.json hbm_gbs",
            "per_launch_ms": round(per_launch_ms, 4), "per_class": per_class}


def traffic_for(kernel):
    """dram read+write bytes per launch from the committed ncu --set full capture, if any."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return d.get(kernel)
    except Exception:
        return None


def oracle_sample(cfg, npoles_sample, seconds_budget=30.0):
    """Time the CPU oracle on a bounded sample: `npoles_sample` of the poles,
    factorization untimed (it is the setup), one resolvent apply each timed;
    the full-step time is extrapolated by the total pole count."""
    from oracle.models import RSW, Wave
    from oracle.rational import build_exp_approx
    from oracle.specelem import Mesh
    m = Mesh(cfg["n"], cfg["p"])
    model = RSW(m, cfg.get("f", 1.0)) if cfg["model"] == "rsw" else Wave(m, make_problem(cfg, m.x, m.y))
    ap = build_exp_approx(cfg["Lambda_tau"], cfg["delta"], verify=False)
    u0 = initial_state(cfg["model"], m.x, m.y, cfg["seed"])
    P = len(ap["poles"])
    idx = np.linspace(0, P - 1, npoles_sample).astype(int)
    solve_s = 0.0
    factor_s = 0.0
    for k in idx:
        t0 = time.perf_counter()
        lu = model.factor(ap["poles"][k] / cfg["tau"])
        factor_s += time.perf_counter() - t0
        t0 = time.perf_counter()
        _ = ap["res"][k] * model.resolvent(ap["poles"][k], cfg["tau"], u0, lu=lu)
        solve_s += time.perf_counter() - t0
    step_s = solve_s / len(idx) * P
    dof = 3 * m.N * cfg["nrhs"]
    return {"value": dof / step_s, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{len(idx)} of {P} poles on the full {cfg['n']}x{cfg['n']}x{cfg['p']}^2 mesh, one "
                      f"resolvent apply each (scipy splu factor untimed, {factor_s:.1f}s), step time "
                      f"extrapolated x{P}/{len(idx)}",
            "step_seconds": step_s}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    res = oracle_sample(cfg, npoles_sample=2)
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["step_seconds"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": args.config, **{k: cfg[k] for k in ("model", "n", "p", "Lambda_tau", "tau",
                                                                      "delta", "nrhs")}},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(time.perf_counter() - t0, 1)}
    print(json.dumps(line), flush=True)


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
    if world > 1:
        # shard the half poles: rank r owns a contiguous range
        tmp = api.setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, device=-1,
                        half_range=(0, 1), **common)
        nh_total = tmp.num_half_poles
        tmp.close()
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
    e = torch.zeros(h.partial_len, dtype=torch.float64, device=dev) if world > 1 else None

    def one_step():
        if world == 1:
            api.apply(h, u, 1)
        else:
            api.step_partial(h, u, e)
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
    if world == 1:
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
    roof = roofline_for(cfg, h, kt, args.steps, pk)
    launches = sum(v[1] for v in kt.values())
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (fp64)", "data": "synthetic",
            "config": {"workload": args.config, "model": cfg["model"], "elements": f"{cfg['n']}x{cfg['n']}",
                       "p": cfg["p"], "Lambda_tau": cfg["Lambda_tau"], "tau": cfg["tau"], "delta": cfg["delta"],
                       "nrhs": cfg["nrhs"], "poles": h.num_poles, "half_poles_total": nh_total,
                       "dof": dof, "nodes_per_field": N,
                       "baseline_nodes_per_field_convention": cfg["n"] ** 2 * cfg["p"] ** 2,
                       "store": "shared" if cfg["model"] == "rsw" else "pernode",
                       "leaf_solver": h.leaf_solver,
                       "merge_kernels": h.stage_report,
                       "store_bytes": h.store_bytes, "work_bytes": h.work_bytes,
                       "l2": "operator store + work buffers exceed the 126 MB L2 (no flush needed)",
                       "parallelism": f"pole-sharded x{world}" if world > 1 else "single GPU"},
            "roofline": roof,
            "kernel_ms": {k: round(v[0], 3) for k, v in kt.items()},
            "gpu_launches": launches, "e2e": e2e,
            "clocks": clk.summary(), "setup_s": round(t_setup, 1), "finite": finite}
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            try:
                cb = oracle_sample(cfg, npoles_sample=2)
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
