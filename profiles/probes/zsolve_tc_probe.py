"""z-solve tile width A/B: 16-column tiles, one CTA per SM (default) against
8-column tiles, two CTAs per SM (ETC_ZTC8=1, a switch of the measured build,
removed after the measurement: profiles/r02/zsolve_tc8_rejected.log)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def run(mode, n, nz, reps=20):
    os.environ["ETC_ZTC8"] = str(mode)
    P.release_plans()
    g = P.GridSpec(n, n, nz, 1.0, 1.0, 1.0)
    rng = np.random.default_rng(5)
    k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, n * n * nz)))
    ds = P.DeviceSystem(P.OrthotropicField(g, *k))
    u = torch.from_numpy(rng.standard_normal(n * n * nz)).cuda()
    out = ds.thomas(u)
    x = out.clone()
    lib = ds.plan.lib
    for _ in range(3): lib.etc_thomas(ds.plan.handle, x.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): lib.etc_thomas(ds.plan.handle, x.data_ptr())
    e1.record(); torch.cuda.synchronize()
    res = out.cpu().numpy()
    del ds
    P.release_plans()
    return res, e0.elapsed_time(e1) / reps

for n, nz in [(128, 128), (256, 256), (512, 512)]:
    a, ta = run(0, n, nz)
    b, tb = run(1, n, nz)
    gb = 16.0 * n * n * nz / 1e9
    print(f"n={n} nz={nz}: bitwise={np.array_equal(a, b)} tc16 {ta:.4f} ms ({gb/ta*1e3:.0f} GB/s) tc8 {tb:.4f} ms ({gb/tb*1e3:.0f} GB/s)", flush=True)
