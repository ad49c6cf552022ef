"""A/B probe: TMA z-solve (ETC_ZTMA=1) vs register-staged k_thomas_x (ETC_ZTMA=0):
bitwise equality of etc_thomas and per-launch time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def run(mode, n, nz, reps=20):
    os.environ["ETC_ZTMA"] = str(mode)
    P.release_plans()
    g = P.GridSpec(n, n, nz, 1.0, 1.0, 1.0)
    rng = np.random.default_rng(5)
    k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, n * n * nz)))
    ds = P.DeviceSystem(P.OrthotropicField(g, *k))
    u = torch.from_numpy(rng.standard_normal(n * n * nz)).cuda()
    out = ds.thomas(u)
    x = out.clone()
    torch.cuda.synchronize()
    lib = ds.plan.lib
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        lib.etc_thomas(ds.plan.handle, x.data_ptr())
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        lib.etc_thomas(ds.plan.handle, x.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return out.cpu().numpy(), ms

for n, nz in [(128, 128), (256, 256), (512, 512), (64, 512), (96, 256)]:
    a, ta = run(0, n, nz)
    b, tb = run(1, n, nz)
    gb = 16.0 * n * n * nz / 1e9
    print(f"n={n} nz={nz}: bitwise={np.array_equal(a, b)} maxrel={np.max(np.abs(a-b))/np.max(np.abs(a)):.3e} "
          f"old {ta:.4f} ms ({gb/ta*1e3:.0f} GB/s)  tma {tb:.4f} ms ({gb/tb*1e3:.0f} GB/s)", flush=True)
