"""N > 1 host logic on CPU (gloo, world size 2): the pole partition covers
every half pole exactly once and the all-reduced partial pole sums reproduce
the single-rank sum.  The per-pole work is done with the oracle here (the CUDA
kernels need a GPU); the decomposition itself is what is tested."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_5168_b200.parallel import half_range


def test_half_range_partition():
    for nh in [1, 7, 168, 282]:
        for world in [1, 2, 3, 8]:
            if nh < world:
                with pytest.raises(ValueError):
                    half_range(nh, 0, world)
                continue
            seen = []
            for r in range(world):
                lo, hi = half_range(nh, r, world)
                assert hi - lo in (nh // world, nh // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(nh))


def _partial_sums(lo, hi):
    """E-like partial sums sum_{m in [lo,hi)} w_m Re(b_m eta_m) computed with the oracle."""
    from oracle.models import RSW
    from oracle.rational import build_exp_approx
    from oracle.specelem import Mesh
    from workloads import rsw_initial_state
    m = Mesh(2, 6)
    model = RSW(m, 1.0)
    tau = 0.2
    ap = build_exp_approx(10.0, 1e-10, verify=False)
    halfs = [(a, b) for a, b in zip(ap["poles"], ap["res"]) if a.imag >= 0]
    u0 = rsw_initial_state(m.x, m.y, 3).real
    E = np.zeros(m.N)
    for k in range(lo, hi):
        a, b = halfs[k]
        w = 2.0 if a.imag > 0 else 1.0
        E += w * (b * model.resolvent(a, tau, u0)[2]).real
    return E, len(halfs)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, nh = _partial_sums(0, 0)
    lo, hi = half_range(nh, rank, world)
    E, _ = _partial_sums(lo, hi)
    t = torch.from_numpy(E)
    dist.all_reduce(t)
    if rank == 0:
        out.put(t.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_partial_sums_reduce_to_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    reduced = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    _, nh = _partial_sums(0, 0)
    full, _ = _partial_sums(0, nh)
    assert np.abs(reduced - full).max() <= 1e-13 * np.abs(full).max()
