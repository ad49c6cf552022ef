"""nz = 1024 z-solve: TMA tiles of 8 columns (k_zsolve_tma<32, double, 8>,
default) against the two-warp register kernel (k_thomas_x2, ETC_Z1024TMA=0):
etc_thomas outputs and time per launch, then the 1024^3 z solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def run(mode, n, nz, reps=10):
    os.environ["ETC_Z1024TMA"] = str(mode)
    P.release_plans()
    g = P.GridSpec(n, n, nz, 1.0, 1.0, 1.0)
    rng = np.random.default_rng(5)
    k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, n * n * nz)))
    ds = P.DeviceSystem(P.OrthotropicField(g, *k))
    u = torch.from_numpy(rng.standard_normal(n * n * nz)).cuda()
    out = ds.thomas(u)
    x = out.clone()
    lib = ds.plan.lib
    for _ in range(2): lib.etc_thomas(ds.plan.handle, x.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): lib.etc_thomas(ds.plan.handle, x.data_ptr())
    e1.record(); torch.cuda.synchronize()
    res = out.cpu().numpy()
    del ds, x, out, u
    P.release_plans()
    return res, e0.elapsed_time(e1) / reps

for n in (64, 256):
    a, ta = run(0, n, 1024)
    b, tb = run(1, n, 1024)
    gb = 16.0 * n * n * 1024 / 1e9
    print(f"n={n} nz=1024: maxrel={np.max(np.abs(a - b)) / np.max(np.abs(a)):.3e} x2 {ta:.4f} ms ({gb / ta * 1e3:.0f} GB/s) "
          f"tma {tb:.4f} ms ({gb / tb * 1e3:.0f} GB/s)", flush=True)
res = {}
for mode in (0, 1):
    os.environ["ETC_Z1024TMA"] = str(mode)
    P.release_plans()
    f = P.gen_random_balls(1024, 40, 0.05, 0.15, 100.0, 11)
    r = P.homogenize(f, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-6)
    res[mode] = r
    print("1024^3 z", mode, r.iterations, "%.15f" % r.kappa_eff, "device s %.3f" % (r.device_ms / 1e3), flush=True)
    del f
    P.release_plans()
    torch.cuda.empty_cache()
