import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1402_5168_b200 import api
from oracle.models import RSW
from oracle.specelem import Mesh
from oracle.rational import build_exp_approx
from workloads import rsw_initial_state
n, p, tau, Lam = 4, 10, 0.2, 100.0
m = Mesh(n, p); model = RSW(m, 1.0)
ap = build_exp_approx(tau*Lam, 1e-10, verify=False)
halfs = [(a, b) for a, b in zip(ap["poles"], ap["res"]) if a.imag >= 0]
u0 = rsw_initial_state(m.x, m.y, 3)
for env in [dict(REXP_LANES="1", REXP_GROUPS="1"), dict()]:
    for k_, v_ in env.items(): os.environ[k_] = v_
    for k in [len(halfs)//2, 5]:
        alpha, b = halfs[k]
        h = api.setup("rsw", n, p, tau, 1e-10, Lam, f=1.0, half_range=(k, k+1))
        u = torch.from_numpy(u0.copy()).reshape(1, 3, -1).cuda()
        e = torch.zeros(h.partial_len, dtype=torch.float64, device="cuda")
        api.step_partial(h, u, e); torch.cuda.synchronize()
        E = e.cpu().numpy().reshape(3, 2, -1)
        w = 2.0 if alpha.imag > 0 else 1.0
        beta = alpha / tau; k2 = beta*beta + 1
        for part, up in enumerate([u0.real.astype(complex), u0.imag.astype(complex)]):
            eta = model.resolvent(alpha, tau, up)[2]
            ref = np.stack([w*(b*eta).real, w*(b*beta/k2*eta).real, w*(-b/k2*eta).real])
            got = E[:, part, :]
            NI = m.NI
            ei = np.linalg.norm(got[:, :NI]-ref[:, :NI])/np.linalg.norm(ref[:, :NI])
            ee = np.linalg.norm(got[:, NI:]-ref[:, NI:])/np.linalg.norm(ref[:, NI:])
            print(env, "pole", k, "part", part, "interior", ei, "edge", ee, "ratio interior", np.linalg.norm(got[:, :NI])/np.linalg.norm(ref[:, :NI]))
        h.close()
