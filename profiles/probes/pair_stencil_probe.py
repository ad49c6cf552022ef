"""A/B probe: two cells per thread along x (k_stencil_pp) vs one
(k_stencil_pht), float64 (ETC_PAIR64) and in the fused float32 solve
(ETC_PAIR32): bitwise operator output (float64), time per launch, solves."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def op64(mode, n, f, reps=30):
    os.environ["ETC_PAIR64"] = str(mode)
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
    rep = P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6)
    rep = P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6)
    return out.cpu().numpy(), ms, rep

for n in (128, 256, 512):
    f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
    a, ta, ra = op64(0, n, f)
    b, tb, rb = op64(1, n, f)
    print(n, "f64 operator bitwise", np.array_equal(a, b), "pht %.4f ms  pp %.4f ms" % (ta, tb),
          "solve it", ra.iterations, rb.iterations, "kappa %.15f %.15f" % (ra.kappa_eff, rb.kappa_eff),
          "ms/it %.3f %.3f" % (ra.device_ms / ra.iterations, rb.device_ms / rb.iterations), flush=True)
os.environ["ETC_PAIR64"] = "0"
for n in (128, 512):
    f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
    res = []
    for m in (0, 1):
        os.environ["ETC_PAIR32"] = str(m)
        P.release_plans()
        P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6, precision="f32")
        r = P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6, precision="f32")
        res.append(r)
    print(n, "f32 single/pair it", res[0].iterations, res[1].iterations, "kappa %.9f %.9f" % (res[0].kappa_eff, res[1].kappa_eff),
          "ms/it %.3f %.3f" % (res[0].device_ms / res[0].iterations, res[1].device_ms / res[1].iterations), flush=True)
