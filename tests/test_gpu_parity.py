"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): relative L2 error <= 1e-10 in complex128 on
identical seeded inputs.  Sizes: BASELINE config 0 in full (every step), a
small variable-coefficient wave case, store modes, nrhs > 1, the pole-sharded
decomposition, edge cases, and at config-1 size (bench launch configuration)
sampled poles against the oracle plus closed-form Fourier evolution.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.evolve import EvolutionOperator  # noqa: E402
from oracle.models import RSW, Wave  # noqa: E402
from oracle.rational import build_exp_approx  # noqa: E402
from oracle.specelem import Mesh  # noqa: E402
from workloads import CONFIGS, rsw_initial_state, wave_initial_state, wave_speed_field  # noqa: E402

TOL = 1e-10


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _api():
    from paper_1402_5168_b200 import api
    return api


def _gpu_apply(h, u0, nsteps):
    u = torch.from_numpy(np.ascontiguousarray(u0)).reshape(h.nrhs, 3, -1).to("cuda")
    _api().apply(h, u, nsteps)
    torch.cuda.synchronize()
    return u.cpu().numpy().reshape(np.shape(u0))


@pytest.fixture(scope="module")
def c0():
    cfg = CONFIGS["c0_rsw_4x4_p10"]
    m = Mesh(cfg["n"], cfg["p"])
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    op = EvolutionOperator(RSW(m, cfg["f"]), cfg["tau"], Lam, cfg["delta"])
    u0 = rsw_initial_state(m.x, m.y, cfg["seed"])
    return cfg, m, op, u0


@pytest.mark.parametrize("store", ["shared", "shared-dense-leaf", "pernode"])
def test_config0_full_run_parity(c0, store, monkeypatch):
    """shared: tensor-product leaf inverse + DMMA GEMMs; shared-dense-leaf: dense q^2 x q^2
    leaf operators (REXP_LEAF=dense); pernode: one operator set per tree node (GEMV path)."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    if store == "shared-dense-leaf":
        monkeypatch.setenv("REXP_LEAF", "dense")
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"],
                     store="pernode" if store == "pernode" else "shared")
    assert h.num_poles == len(op.poles)
    nst = cfg["nsteps"] if store != "pernode" else 3
    got = _gpu_apply(h, u0, nst)
    ref = op.evolve(u0, nst)
    err = rel_l2(got, ref)
    print(f"config0 {store} {nst} steps rel L2 {err:.3e}")
    assert err <= TOL
    h.close()


def test_config0_nrhs2_and_host_path(c0):
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    u1 = rsw_initial_state(m.x, m.y, cfg["seed"] + 1)
    U = np.stack([u0, u1])
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=2)
    got = _gpu_apply(h, U, 2)
    for k, uk in enumerate([u0, u1]):
        assert rel_l2(got[k], op.evolve(uk, 2)) <= TOL
    # host-pointer path gives the same bits as the device path
    Uh = np.ascontiguousarray(U.copy())
    _api().apply(h, Uh, 2)
    assert np.array_equal(Uh, got)
    h.close()


@pytest.mark.parametrize("nrhs,chunk", [(8, "37"), (3, "1000"), (4, "1000")])
def test_config0_many_rhs_and_pole_chunks(c0, nrhs, chunk, monkeypatch):
    """Multi-RHS path (config 3's shape at config 0 size): nrhs independent states,
    runtime-R2 DMMA GEMMs at every level incl. the periodic closure, and the pole
    sums accumulated over chunks of half poles (REXP_CHUNK)."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    monkeypatch.setenv("REXP_CHUNK", chunk)
    U = np.stack([rsw_initial_state(m.x, m.y, cfg["seed"] + 10 * k) for k in range(nrhs)])
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=nrhs)
    got = _gpu_apply(h, U, 2)
    errs = [rel_l2(got[k], op.evolve(U[k], 2)) for k in range(nrhs)]
    print(f"nrhs {nrhs} chunk {chunk}: max rel L2 {max(errs):.3e}")
    assert max(errs) <= TOL
    h.close()


@pytest.mark.parametrize("lanes,chunk,graph", [("1", "1000", "1"), ("3", "23", "1"), ("2", "1000", "0")])
def test_config0_lanes_chunks_graph(c0, lanes, chunk, graph, monkeypatch):
    """Execution modes of the shared store: pole lanes on forked streams
    (REXP_LANES), pole chunks inside each lane with per-lane accumulation of the
    spectral pole sums (REXP_CHUNK), CUDA-graph replay vs eager launches
    (REXP_GRAPH).  Every mode matches the oracle; graph replay and eager
    launches give identical bits (same kernels, no atomics)."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    monkeypatch.setenv("REXP_LANES", lanes)
    monkeypatch.setenv("REXP_CHUNK", chunk)
    monkeypatch.setenv("REXP_GRAPH", graph)
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
    got = _gpu_apply(h, u0, 3)
    err = rel_l2(got, op.evolve(u0, 3))
    print(f"lanes {lanes} chunk {chunk} graph {graph}: rel L2 {err:.3e}")
    assert err <= TOL
    h.close()
    # bitwise: the same stage configuration (no autotuning: a GEMV and a GEMM sum
    # in different orders), graph replay vs eager launches
    monkeypatch.setenv("REXP_AUTOTUNE", "0")
    outs = []
    for g in ("1", "0"):
        monkeypatch.setenv("REXP_GRAPH", g)
        h2 = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
        outs.append(_gpu_apply(h2, u0, 3))
        h2.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("nrhs", [1, 3])
def test_config0_three_stage_gemm(c0, nrhs, monkeypatch):
    """The 3-stage cp.async merge GEMM (an autotuner candidate) forced on every
    GEMM stage of the up-Y and down sweeps (REXP_GEMM_STAGES=3), compile-time
    and runtime R2."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    monkeypatch.setenv("REXP_GEMM_STAGES", "3")
    U = np.stack([rsw_initial_state(m.x, m.y, cfg["seed"] + 10 * k) for k in range(nrhs)])
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=nrhs)
    assert "s3" in h.stage_report
    got = _gpu_apply(h, U, 2)
    errs = [rel_l2(got[k], op.evolve(U[k], 2)) for k in range(nrhs)]
    print(f"3-stage GEMM nrhs {nrhs}: max rel L2 {max(errs):.3e}")
    assert max(errs) <= TOL
    h.close()


@pytest.mark.parametrize("nrhs,stages", [(8, "tuned"), (8, "3"), (64, "tuned"), (64, "x1")])
def test_config0_symmetric_pair_gemm_many_rhs(c0, nrhs, stages, monkeypatch):
    """nrhs = 8 (R2 = 16, runtime R2) and 64 (R2 = 128, config 3's RHS count,
    compile-time R2): every merge level above the first runs as the
    symmetric-pair DMMA GEMM (k_cgemm_sym) or GEMV; "3" forces the 3-stage
    cp.async variant on its up-Y / down stages; parity per RHS (every
    (nrhs/8)-th RHS against the oracle: the RHS are independent)."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    if stages in ("3", "x1"):   # "x1": the single-stage cp.async ring of the up-X pair GEMM (R2 = 128)
        monkeypatch.setenv("REXP_GEMM_STAGES", stages)
    U = np.stack([rsw_initial_state(m.x, m.y, cfg["seed"] + 10 * k) for k in range(nrhs)])
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=nrhs)
    assert "symgemm" in h.stage_report
    if stages == "3":
        assert "s3" in h.stage_report
    if stages == "x1":
        assert "s1" in h.stage_report
    got = _gpu_apply(h, U, 2)
    errs = [rel_l2(got[k], op.evolve(U[k], 2)) for k in range(0, nrhs, nrhs // 8)]
    print(f"symmetric-pair GEMM nrhs {nrhs}: max rel L2 {max(errs):.3e}")
    assert max(errs) <= TOL
    h.close()


@pytest.mark.parametrize("nrhs,up,down", [(1, "2", "2"), (2, "2", "0"), (4, "0", "2"), (8, "2", "2"), (64, "2", "2"),
                                          (8, "3", "3"), (4, "3", "3")])
def test_config0_fused_subtree_sweeps(c0, nrhs, up, down, monkeypatch):
    """The fused multi-level merge kernels (fused_tree.cu: boundary data of a
    subtree resident in shared memory, operators streamed by bulk copies on
    mbarriers) forced on (REXP_FUSE_FORCE keeps them even where the autotuner
    would prefer the single-level launches): levels (1, 2) upward and (2, 1)
    downward, separately and together, and all three levels of config 0's tree in
    one kernel; column layouts RC = 2, 4, 8 (R2 = 2, 4, 8 and wider)."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    monkeypatch.setenv("REXP_FUSE_UP", up)
    monkeypatch.setenv("REXP_FUSE_DOWN", down)
    monkeypatch.setenv("REXP_FUSE_FORCE", "1")
    if nrhs >= 8:   # the fused kernels read the half-pair operator layout (no second reflection)
        monkeypatch.setenv("REXP_NO_SYM2", "1")
    U = np.stack([rsw_initial_state(m.x, m.y, cfg["seed"] + 10 * k) for k in range(nrhs)])
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=nrhs)
    rep = h.stage_report
    assert ("fused_up" in rep) == (up != "0") and ("fused_down" in rep) == (down != "0"), rep
    got = _gpu_apply(h, U, 2)
    ks = range(0, nrhs, max(1, nrhs // 4))
    errs = [rel_l2(got[k], op.evolve(U[k], 2)) for k in ks]
    print(f"fused sweeps nrhs {nrhs} up {up} down {down}: max rel L2 {max(errs):.3e}")
    assert max(errs) <= TOL
    h.close()


def test_config0_long_run_accumulation(c0):
    """60 steps (graph replay, pole lanes): the error against the oracle must not
    grow beyond the per-step rounding (no drift from the spectral / pair /
    Fourier re-expressions).  The plain vector 2-norm is not the discrete energy
    (L is skew only in a quadrature-weighted inner product), so its change is
    compared with the oracle's rather than with 1."""
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
    got = _gpu_apply(h, u0, 60)
    ref = op.evolve(u0, 60)
    err = rel_l2(got, ref)
    growth = float(np.linalg.norm(got) / np.linalg.norm(u0))
    growth_ref = float(np.linalg.norm(ref) / np.linalg.norm(u0))
    print(f"config0 60 steps rel L2 {err:.3e}, norm ratio {growth:.6f} (oracle {growth_ref:.6f})")
    assert err <= TOL
    assert abs(growth - growth_ref) <= 1e-10
    h.close()


def test_edge_cases_zero_state_and_zero_steps(c0):
    cfg, m, op, u0 = c0
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
    assert np.array_equal(_gpu_apply(h, u0, 0), u0)
    z = np.zeros_like(u0)
    assert np.array_equal(_gpu_apply(h, z, 3), z)
    # real input stays real (conjugate-pair evaluation is exactly real)
    ur = u0.real.astype(complex)
    out = _gpu_apply(h, ur, 2)
    assert np.abs(out.imag).max() == 0.0
    h.close()


def test_wave_variable_kappa_parity():
    n, p, tau, Lam = 4, 10, 0.2, 100.0
    m = Mesh(n, p)
    kappa = wave_speed_field(m.x, m.y, seed=11)
    u0 = wave_initial_state(m.x, m.y, seed=5)
    op = EvolutionOperator(Wave(m, kappa), tau, Lam, 1e-10)
    h = _api().setup("wave", n, p, tau, 1e-10, Lam, kappa=kappa)
    got = _gpu_apply(h, u0, 3)
    err = rel_l2(got, op.evolve(u0, 3))
    print(f"wave rel L2 {err:.3e}")
    assert err <= TOL
    h.close()


def test_ragged_small_mesh_p4_and_p18():
    """Smallest element order (p=4, 2x2 leaves of 2x2) and the largest this build allows."""
    for n, p in [(2, 4), (2, 18)]:
        m = Mesh(n, p)
        u0 = rsw_initial_state(m.x, m.y, seed=3)
        op = EvolutionOperator(RSW(m, 1.0), 0.1, 100.0, 1e-10)
        h = _api().setup("rsw", n, p, 0.1, 1e-10, 100.0, f=1.0)
        err = rel_l2(_gpu_apply(h, u0, 2), op.evolve(u0, 2))
        assert err <= TOL, (n, p, err)
        h.close()


def test_pole_sharded_decomposition_equals_full(c0):
    """Multi-GPU decomposition (PAPER.md:139-140 'all the inverse operators ... can be
    applied independently'): two handles owning disjoint half-pole ranges, partial pole
    sums added, then finish == single-handle apply (same device, sequential)."""
    cfg, m, op, u0 = c0
    api = _api()
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    full = api.setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
    nh = full.num_half_poles
    ha = api.setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], half_range=(0, nh // 3))
    hb = api.setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], half_range=(nh // 3, nh))
    u = torch.from_numpy(u0.copy()).reshape(1, 3, -1).cuda()
    ea = torch.zeros(ha.partial_len, dtype=torch.float64, device="cuda")
    eb = torch.zeros_like(ea)
    api.step_partial(ha, u, ea)
    api.step_partial(hb, u, eb)
    api.step_finish(ha, ea + eb, u)
    torch.cuda.synchronize()
    ref = _gpu_apply(full, u0, 1)
    got = u.cpu().numpy().reshape(3, -1)
    assert rel_l2(got, ref) <= 1e-13
    for hh in (full, ha, hb):
        hh.close()


# --------------------------------------------------------------------------
# BASELINE config 1 size, bench launch configuration
# --------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c1_handle():
    cfg = CONFIGS["c1_rsw_16x16_p16"]
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"])
    yield cfg, h
    h.close()


def test_config1_fourier_mode_closed_form(c1_handle):
    """Property at full size: a resolved Fourier mode evolves by expm(tau * symbol)
    (PAPER.md:941-946), independent of the oracle."""
    cfg, h = c1_handle
    x, y = h.node_coords()
    k = (2, -3)
    vec = np.array([0.3 - 0.1j, -0.2, 1.0 + 0.5j])
    ph = np.exp(2j * math.pi * (k[0] * x + k[1] * y))
    u0 = vec[:, None] * ph[None, :]
    a1, a2 = 2j * math.pi * k[0], 2j * math.pi * k[1]
    f = cfg["f"]
    S = np.array([[0, -f, a1], [f, 0, a2], [a1, a2, 0]], dtype=complex)
    got = _gpu_apply(h, u0, 4)
    ref = sla.expm(4 * cfg["tau"] * S) @ vec
    err = np.abs(got - ref[:, None] * ph[None, :]).max() / np.abs(vec).max()
    print(f"config1 Fourier-mode 4-step error {err:.3e}")
    assert err <= 1e-9


def test_config1_sampled_poles_against_oracle(c1_handle):
    """Sampled outputs at full size: single-pole partial sums from the bench's kernels
    (same grid shapes, grid.y = 1) vs the oracle's sparse solve of that pole."""
    cfg, h = c1_handle
    api = _api()
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    tau, f = cfg["tau"], cfg["f"]
    m = Mesh(cfg["n"], cfg["p"])
    model = RSW(m, f)
    ref_ap = build_exp_approx(cfg["Lambda_tau"], cfg["delta"], verify=False)
    halfs = [(a, b) for a, b in zip(ref_ap["poles"], ref_ap["res"]) if a.imag >= 0]
    u0 = rsw_initial_state(m.x, m.y, cfg["seed"])
    ur = u0.real
    # sample the poles that matter: the largest residue and one ~1e-2 of it (outer
    # filter poles have |b| ~ 1e-15, where residues agree only in absolute terms)
    mags = np.array([abs(b) for _, b in halfs])
    k_big = int(np.argmax(mags))
    k_mid = int(np.argmin(np.abs(mags - 1e-2 * mags.max())))
    for k in [k_big, k_mid]:
        alpha, b = halfs[k]
        w = 2.0 if alpha.imag > 0 else 1.0
        hk = api.setup("rsw", cfg["n"], cfg["p"], tau, cfg["delta"], Lam, f=f, half_range=(k, k + 1))
        u = torch.from_numpy(u0.copy()).reshape(1, 3, -1).cuda()
        e = torch.zeros(hk.partial_len, dtype=torch.float64, device="cuda")
        api.step_partial(hk, u, e)
        torch.cuda.synchronize()
        E = e.cpu().numpy().reshape(3, 2, -1)       # [nE][R2][N]; R2 part 0 = Re(u0)
        r = model.resolvent(alpha, tau, ur)          # oracle (tau L - alpha)^{-1} Re(u0)
        eta = r[2]
        beta = alpha / tau
        k2 = beta * beta + f * f
        pp, qq = beta / k2, -f / k2
        ref = np.stack([w * (b * eta).real, w * (b * pp * eta).real, w * (b * qq * eta).real])
        err = rel_l2(E[:, 0, :], ref)
        print(f"config1 half pole {k} rel L2 {err:.3e}")
        assert err <= TOL
        hk.close()


def test_config3_many_rhs_fourier_modes_closed_form():
    """BASELINE config 3 (32x32 elements, p = 16, 64 RHS) in the bench's launch
    configuration: every RHS is a different resolved Fourier mode, each checked
    against expm(tau * symbol) after 2 steps."""
    cfg = CONFIGS["c3_rsw_32x32_p16_x64"]
    Lam = cfg["Lambda_tau"] / cfg["tau"]
    h = _api().setup("rsw", cfg["n"], cfg["p"], cfg["tau"], cfg["delta"], Lam, f=cfg["f"], nrhs=cfg["nrhs"])
    x, y = h.node_coords()
    rng = np.random.default_rng(9)
    U, refs = [], []
    f = cfg["f"]
    for k in range(cfg["nrhs"]):
        k1, k2 = (int(v) for v in rng.integers(-5, 6, size=2))
        vec = rng.standard_normal(3) + 1j * rng.standard_normal(3)
        ph = np.exp(2j * math.pi * (k1 * x + k2 * y))
        a1, a2 = 2j * math.pi * k1, 2j * math.pi * k2
        S = np.array([[0, -f, a1], [f, 0, a2], [a1, a2, 0]], dtype=complex)
        U.append(vec[:, None] * ph[None, :])
        refs.append((sla.expm(2 * cfg["tau"] * S) @ vec)[:, None] * ph[None, :])
    got = _gpu_apply(h, np.stack(U), 2)
    err = max(np.abs(got[k] - refs[k]).max() / np.abs(refs[k]).max() for k in range(cfg["nrhs"]))
    print(f"config3 64-RHS Fourier-mode 2-step max error {err:.3e}")
    assert err <= 1e-9
    h.close()
