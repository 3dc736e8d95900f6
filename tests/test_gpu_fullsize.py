"""GPU parity at the sizes the bench runs, against committed oracle outputs.

The golden files under tests/golden/ are written by tests/golden/make_golden.py,
which calls only oracle/ (EvolutionOperator.step over ALL poles, or one
EvolutionOperator.resolvent).  Bar (BASELINE.json north_star): relative L2
error <= 1e-10 in complex128 on identical seeded inputs.

  * config 1 (16x16 elements, p = 16): steps 1 and 3 in full, the bench's
    handle (pole lanes, autotuned merge stages, CUDA-graph replay);
  * config 3 (32x32, p = 16, 64 RHS): one step, RHS 0/21/42/63 at 16384
    sampled nodes (all three fields) plus each RHS's full output norm;
  * c2r (per-node wave store at q = 14): three steps in full;
  * configs 2 and 4 at full mesh, pole-sharded handles: the pole sums of two
    sampled half poles (one rank's work of the sharded run) against the
    oracle's resolvent of that pole;
  * n = 4, p = 16 full runs against the live oracle (the q = 14 kernel
    instantiations at a size the oracle finishes in seconds), RSW and wave,
    and the per-node store with nrhs = 2 and 4.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.evolve import EvolutionOperator  # noqa: E402
from oracle.models import RSW, Wave  # noqa: E402
from oracle.specelem import Mesh  # noqa: E402
from workloads import CONFIGS, initial_state, rsw_initial_state, wave_initial_state, wave_speed_field  # noqa: E402

TOL = 1e-10
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _api():
    from paper_1402_5168_b200 import api
    return api


def _golden(name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.fail(f"missing golden file {name}: run tests/golden/make_golden.py")
    return np.load(path)


def _setup(cfg, **kw):
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    kappa = None
    if cfg["model"] == "wave":
        x, y = _api().mesh_coords(cfg["n"], cfg["p"])
        kappa = wave_speed_field(x, y, cfg["seed"])
    return _api().setup(cfg["model"], cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg.get("f", 1.0),
                        kappa=kappa, **kw)


def _check_poles(h, g):
    """The handle's poles/weights are the oracle's (C++ and Python share no code)."""
    a, b = h.poles()
    assert len(a) == len(g["poles"])
    assert np.abs(a - g["poles"]).max() <= 1e-12 * np.abs(g["poles"]).max()
    assert np.abs(b - g["res"]).max() <= 1e-12 * np.abs(g["res"]).max()


def _to_dev(U):
    return torch.from_numpy(np.ascontiguousarray(U)).to("cuda")


@pytest.mark.parametrize("case", ["c1", "c2r"])
def test_full_steps_against_golden(case):
    g = _golden(f"{case}_steps.npz")
    cfg = CONFIGS[str(g["config"])]
    h = _setup(cfg, nrhs=1)
    _check_poles(h, g)
    x, y = h.node_coords()
    u0 = initial_state(cfg["model"], x, y, cfg["seed"])
    assert rel_l2(u0, g["u0"]) <= 1e-14          # the same seeded input on both sides
    u = _to_dev(g["u0"][None])
    errs = []
    for s in (1, 2, 3):
        _api().apply(h, u, 1)
        torch.cuda.synchronize()
        got = u.cpu().numpy()[0]
        errs.append(rel_l2(got, g[f"u{s}"]))
    print(f"{case}: rel L2 after steps 1..3 = " + ", ".join(f"{e:.2e}" for e in errs) + f" ({h.stage_report})")
    h.close()
    assert max(errs) <= TOL


def test_config3_sampled_rhs_against_golden():
    """Full config-3 step for sampled RHS.  Its golden needs all 528 sparse LU
    factorizations of the 32x32 mesh (~90 s and ~4 GB each: ~14 CPU-hours), so
    it is generated on demand (tests/golden/make_golden.py c3) and the test is
    skipped while the file is absent; the committed full-size check of the 64-RHS
    kernels is test_config3_full_mesh_sampled_poles_64rhs_against_golden."""
    if not os.path.exists(os.path.join(GOLD, "c3_step1_sampled.npz")):
        pytest.skip("c3_step1_sampled.npz not generated (~14 CPU-hours of oracle LU factorizations)")
    g = _golden("c3_step1_sampled.npz")
    cfg = CONFIGS[str(g["config"])]
    h = _setup(cfg, nrhs=cfg["nrhs"])
    _check_poles(h, g)
    x, y = h.node_coords()
    U = np.stack([rsw_initial_state(x, y, cfg["seed"] + 10 * k) for k in range(cfg["nrhs"])])
    u = _to_dev(U)
    _api().apply(h, u, 1)
    torch.cuda.synchronize()
    got = u.cpu().numpy()
    idx = g["idx"]
    errs, nerrs = [], []
    for j, k in enumerate(g["rhs"]):
        errs.append(rel_l2(got[k][:, idx], g["u1"][j]))
        nerrs.append(abs(np.linalg.norm(got[k]) - g["norm"][j]) / g["norm"][j])
    print(f"config3 sampled RHS {list(g['rhs'])}: rel L2 {max(errs):.2e}, norm {max(nerrs):.2e}")
    h.close()
    assert max(errs) <= TOL and max(nerrs) <= TOL


def _pole_sum_reference(model, alpha, b, tau, f, R):
    """This half pole's pole sums E_k formed from the oracle's
    resolvent R = (tau L - alpha)^{-1} u_part of the real / imaginary parts of
    u0 ([part][field][node]): weight 2 (1 for a real pole) times
    Re(d_k x); RSW d = (b, b p, b q) on eta with A_beta = p I + q J,
    wave d = (b, b / beta) on v (the (1/tau) of reading R9 is inside R)."""
    w = 2.0 if alpha.imag > 0 else 1.0
    beta = alpha / tau
    if model == "rsw":
        k2 = beta * beta + f * f
        ds = [b, b * beta / k2, -b * f / k2]
    else:
        ds = [b, b / beta]
    return np.stack([np.stack([w * (d * R[part][2]).real for part in range(2)]) for d in ds])


@pytest.mark.parametrize("case", ["c2s", "c4s"])
def test_full_mesh_shard_pole_sums_against_golden(case):
    """Configs 2 and 4 (full meshes) through the pole-sharded entry point
    (rexp_step_partial): a handle owning one sampled half pole, its pole sums
    against the oracle's resolvent of that pole at sampled nodes."""
    g = _golden(f"{case}_poles_sampled.npz")
    cfg = CONFIGS[str(g["config"])]
    x, y = _api().mesh_coords(cfg["n"], cfg["p"])
    u0 = initial_state(cfg["model"], x, y, cfg["seed"])
    idx = g["idx"]
    for j, k in enumerate(g["half_index"]):
        h = _setup(cfg, nrhs=1, half_range=(int(k), int(k) + 1))
        _check_poles(h, g)
        u = _to_dev(u0[None])
        e = torch.zeros(h.partial_len, dtype=torch.float64, device="cuda")
        _api().step_partial(h, u, e)
        torch.cuda.synchronize()
        nE = 3 if cfg["model"] == "rsw" else 2
        E = e.cpu().numpy().reshape(nE, 2, -1)[:, :, idx]
        fi = int(g["full_index"][j])
        ref = _pole_sum_reference(cfg["model"], g["poles"][fi], g["res"][fi], cfg["tau"], cfg.get("f", 1.0),
                                  g["R"][j])
        err = rel_l2(E, ref)
        print(f"{case} half pole {k}: pole sums rel L2 {err:.2e} (store {h.store_bytes / 1e9:.2f} GB)")
        h.close()
        assert err <= TOL


def test_config3_full_mesh_sampled_poles_64rhs_against_golden():
    """Config 3 at full size through the 64-RHS (R2 = 128) kernels: a handle
    owning one sampled half pole applies it to all 64 seeded right-hand sides;
    the pole sums of the first and the last RHS against the oracle's resolvent
    of that pole (sampled nodes).  Pole by pole the comparison is free of the
    cancellation in sum_m b_m R_m u (sum |b_m| = 2.8e3, R15)."""
    g = _golden("c3s_poles_sampled.npz")
    cfg = CONFIGS[str(g["config"])]
    x, y = _api().mesh_coords(cfg["n"], cfg["p"])
    U = np.stack([rsw_initial_state(x, y, cfg["seed"] + 10 * k) for k in range(cfg["nrhs"])])
    idx = g["idx"]
    for j, k in enumerate(g["half_index"]):
        h = _setup(cfg, nrhs=cfg["nrhs"], half_range=(int(k), int(k) + 1))
        _check_poles(h, g)
        u = _to_dev(U)
        e = torch.zeros(h.partial_len, dtype=torch.float64, device="cuda")
        _api().step_partial(h, u, e)
        torch.cuda.synchronize()
        E = e.cpu().numpy().reshape(3, 2 * cfg["nrhs"], -1)[:, :, idx]
        fi = int(g["full_index"][j])
        errs = []
        for t, r in enumerate(g["rhs"]):
            ref = _pole_sum_reference("rsw", g["poles"][fi], g["res"][fi], cfg["tau"], cfg["f"], g["R"][j][2 * t:2 * t + 2])
            errs.append(rel_l2(E[:, 2 * r:2 * r + 2], ref))
        print(f"c3s half pole {k}: pole sums of RHS {list(g['rhs'])} rel L2 {max(errs):.2e} ({h.stage_report[:80]})")
        h.close()
        assert max(errs) <= TOL


# --------------------------------------------------------------------------
# q = 14 kernel instantiations at a size the live oracle finishes in seconds
# --------------------------------------------------------------------------
def test_rsw_n4_p16_full_run_live_oracle():
    n, p, tau, Lam = 4, 16, 0.25, 80.0
    m = Mesh(n, p)
    U = np.stack([rsw_initial_state(m.x, m.y, 21 + 10 * k) for k in range(2)])
    op = EvolutionOperator(RSW(m, 1.0), tau, Lam, 1e-10)
    for nrhs in (1, 2):
        h = _api().setup("rsw", n, p, tau, 1e-10, Lam, f=1.0, nrhs=nrhs)
        assert h.leaf_solver == "spectral"
        u = _to_dev(U[:nrhs])
        _api().apply(h, u, 3)
        torch.cuda.synchronize()
        got = u.cpu().numpy()
        errs = [rel_l2(got[k], op.evolve(U[k], 3)) for k in range(nrhs)]
        print(f"rsw n4 p16 nrhs {nrhs}: rel L2 {max(errs):.2e}")
        h.close()
        assert max(errs) <= TOL


@pytest.mark.parametrize("nrhs", [1, 2, 4])
def test_wave_pernode_q14_and_nrhs_live_oracle(nrhs):
    """Per-node (variable kappa) store: q = 14 leaves (n = 4, p = 16) for one
    RHS, and nrhs = 2 / 4 (the batched leaf GEMVs launch_leaf_up_nb<4/8>)."""
    n, p, tau, Lam = (4, 16, 0.2, 100.0) if nrhs == 1 else (4, 10, 0.2, 100.0)
    m = Mesh(n, p)
    kappa = wave_speed_field(m.x, m.y, seed=11)
    U = np.stack([wave_initial_state(m.x, m.y, 5 + 10 * k) for k in range(nrhs)])
    op = EvolutionOperator(Wave(m, kappa), tau, Lam, 1e-10)
    h = _api().setup("wave", n, p, tau, 1e-10, Lam, kappa=kappa, nrhs=nrhs)
    u = _to_dev(U)
    _api().apply(h, u, 2)
    torch.cuda.synchronize()
    got = u.cpu().numpy()
    errs = [rel_l2(got[k], op.evolve(U[k], 2)) for k in range(nrhs)]
    print(f"wave pernode n{n} p{p} nrhs {nrhs}: rel L2 {max(errs):.2e}")
    h.close()
    assert max(errs) <= TOL
