#!/usr/bin/env python
"""Write the full-size golden outputs the GPU parity tests compare against.

Calls ONLY ``oracle/`` (and the seeded input generators of ``workloads.py``):
every stored value is ``oracle.evolve.EvolutionOperator.step`` (the plain
definition  u_{n+1} = sum_m b_m (tau L - alpha_m)^{-1} u_n  over ALL poles,
PAPER.md:61-65) or one ``EvolutionOperator.resolvent`` (one pole,
PAPER.md:58-60).  Nothing here reads the CUDA path.

The only liberty taken is parallelism: the per-pole terms b_m R_m u of one
step are computed in a process pool (one sparse LU per pole, freed after use:
a config-3 factor is ~4 GB) and summed in the main process in ascending m,
exactly the order of ``EvolutionOperator.step``.

    python tests/golden/make_golden.py c1 c2r c3 [--procs 8]

Cases (DESIGN.md §9 "Full-size parity"):
  c1   BASELINE config 1, 3 steps from the seeded state: u1 and u3 in full.
  c2r  reduced wave config (per-node store, q = 14), 3 steps: u1..u3 in full.
  c3   BASELINE config 3, one step of RHS k in {0, 21, 42, 63} (seed + 10k) at
       16384 sampled nodes (all three fields) + each RHS's full output norm.
  c2s, c4s  BASELINE configs 2 and 4 at full mesh: the resolvent of two
       sampled half poles applied to Re(u0) and Im(u0), at sampled nodes (the
       pole-sharded GPU runs are checked pole by pole).
  c3s  BASELINE config 3 at full mesh: the same two-sampled-half-pole
       resolvents for the first and the last of the 64 right-hand sides
       (seed + 10k, k = 0 and 63): the 64-RHS (R2 = 128) kernels pole by pole.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))

from oracle.evolve import EvolutionOperator  # noqa: E402
from oracle.models import RSW, Wave  # noqa: E402
from oracle.specelem import Mesh  # noqa: E402
from workloads import CONFIGS, initial_state, wave_speed_field  # noqa: E402

NSAMPLE = 16384
CASES = {
    "c1": "c1_rsw_16x16_p16",
    "c2r": "c2r_wave_8x8_p16",
    "c3": "c3_rsw_32x32_p16_x64",
    "c2s": "c2_wave_32x32_p16",
    "c4s": "c4_wave_64x64_p12",
    "c3s": "c3_rsw_32x32_p16_x64",
}

_G = {}


def make_op(cfg):
    m = Mesh(cfg["n"], cfg["p"])
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    if cfg["model"] == "rsw":
        model = RSW(m, cfg["f"])
    else:
        model = Wave(m, wave_speed_field(m.x, m.y, cfg["seed"]))
    return m, EvolutionOperator(model, cfg["tau"], Lam, cfg["delta"])


def _init(cfg):
    _G["m"], _G["op"] = make_op(cfg)


def _term(args):
    """b_m (tau L - alpha_m)^{-1} u for every state u in the file (one LU, then freed)."""
    m_idx, path = args
    op = _G["op"]
    U = np.load(path)
    out = np.stack([op.res[m_idx] * op.resolvent(m_idx, u) for u in U])
    op._lu[m_idx] = None
    return m_idx, out


def _resolvent_only(args):
    """(tau L - alpha_m)^{-1} u (no weight) for every state u in the file."""
    m_idx, path = args
    op = _G["op"]
    U = np.load(path)
    out = np.stack([op.resolvent(m_idx, u) for u in U])
    op._lu[m_idx] = None
    return m_idx, out


def steps(pool, op, U, nsteps, tag):
    """nsteps of EvolutionOperator.step applied to every state in U (pole-parallel)."""
    outs = []
    for s in range(nsteps):
        path = f"/tmp/golden_{tag}_in{s}.npy"
        np.save(path, U)
        acc = np.zeros_like(U)
        t0 = time.time()
        expect = 0
        for m_idx, term in pool.imap(_term, [(k, path) for k in range(len(op.poles))], chunksize=1):
            assert m_idx == expect
            expect += 1
            acc += term               # ascending m, as EvolutionOperator.step
        print(f"[{tag}] step {s + 1}/{nsteps}: {len(op.poles)} poles in {time.time() - t0:.0f}s", flush=True)
        os.remove(path)
        U = acc
        outs.append(U.copy())
    return outs


def run(case, procs):
    import multiprocessing as mp
    name = CASES[case]
    cfg = CONFIGS[name]
    m, op = make_op(cfg)
    meta = dict(config=name, poles=op.poles, res=op.res, N=m.N)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_init, initargs=(cfg,)) as pool:
        if case in ("c1", "c2r"):
            U0 = initial_state(cfg["model"], m.x, m.y, cfg["seed"])[None]
            outs = steps(pool, op, U0, 3, case)
            np.savez(os.path.join(HERE, f"{case}_steps.npz"), u0=U0[0], u1=outs[0][0], u2=outs[1][0],
                     u3=outs[2][0], **meta)
        elif case == "c3":
            ks = [0, 21, 42, 63]
            U0 = np.stack([initial_state("rsw", m.x, m.y, cfg["seed"] + 10 * k) for k in ks])
            (u1,) = steps(pool, op, U0, 1, case)
            idx = np.sort(np.random.default_rng(20260).choice(m.N, NSAMPLE, replace=False))
            np.savez(os.path.join(HERE, "c3_step1_sampled.npz"), rhs=np.array(ks), idx=idx,
                     u1=u1[:, :, idx], norm=np.linalg.norm(u1.reshape(len(ks), -1), axis=1), **meta)
        else:
            # sampled half poles: the largest |b| and one ~1e-2 of it
            half = [k for k in range(len(op.poles)) if op.poles[k].imag >= 0]
            mags = np.array([abs(op.res[k]) for k in half])
            picks = [int(np.argmax(mags)), int(np.argmin(np.abs(mags - 1e-2 * mags.max())))]
            rhs = [0, cfg["nrhs"] - 1] if case == "c3s" else [0]
            meta["rhs"] = np.array(rhs)
            parts = []
            for k in rhs:
                u0 = initial_state(cfg["model"], m.x, m.y, cfg["seed"] + 10 * k)
                parts += [u0.real.astype(complex), u0.imag.astype(complex)]
            parts = np.stack(parts)
            path = f"/tmp/golden_{case}_parts.npy"
            np.save(path, parts)
            res = dict(pool.imap(_resolvent_only, [(half[j], path) for j in picks], chunksize=1))
            idx = np.sort(np.random.default_rng(20261).choice(m.N, NSAMPLE, replace=False))
            np.savez(os.path.join(HERE, f"{case}_poles_sampled.npz"), half_index=np.array(picks),
                     full_index=np.array([half[j] for j in picks]), idx=idx,
                     R=np.stack([res[half[j]][:, :, idx] for j in picks]), **meta)
    print(f"[{case}] written", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+", choices=sorted(CASES))
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    for c in a.cases:
        run(c, a.procs)


if __name__ == "__main__":
    main()
