"""A/B probe of a float64 phase-stencil switch: python stencil_env_ab.py VAR A B
-> bitwise operator output, ms per operator launch, and the 512^3 z solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

var, vals = sys.argv[1], sys.argv[2:]

def run(v, n, f, reps=30):
    os.environ[var] = v
    P.release_plans()
    ds = P.DeviceSystem(f)
    torch.manual_seed(0)
    u = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
    out = ds.apply_operator(u)
    y = torch.empty_like(u)
    lib, h = ds.plan.lib, ds.plan.handle
    for _ in range(3): lib.etc_apply_operator(h, u.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): lib.etc_apply_operator(h, u.data_ptr(), y.data_ptr())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del ds
    P.release_plans()
    P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6)
    rep = P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6)
    return out.cpu().numpy(), ms, rep

for n in (128, 256, 512):
    f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
    res = [run(v, n, f) for v in vals]
    print(n, var, vals, "operator bitwise", all(np.array_equal(res[0][0], r[0]) for r in res[1:]),
          "ms", ["%.4f" % r[1] for r in res], "it", [r[2].iterations for r in res],
          "kappa", ["%.15f" % r[2].kappa_eff for r in res], "ms/it", ["%.3f" % (r[2].device_ms / r[2].iterations) for r in res],
          flush=True)
