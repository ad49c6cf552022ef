"""cluster (ETC_QPLANES=0) vs decoupled (1) plane transforms: bitwise + time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P
def run(mode, n, reps=20):
    os.environ["ETC_QPLANES"] = str(mode)
    P.release_plans()
    g = P.GridSpec(n, n, n, 1.0, 1.0, 1.0)
    ds = P.DeviceSystem(P.OrthotropicField(g, *np.ones((3, n ** 3))))
    torch.manual_seed(0)
    x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    lib, h = ds.plan.lib, ds.plan.handle
    outs, times = [], []
    for fn in (lib.etc_dct2_xy, lib.etc_dct3_xy, lib.etc_apply_precond):
        fn(h, x.data_ptr(), y.data_ptr()); torch.cuda.synchronize()
        outs.append(y.cpu().numpy().copy())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3): fn(h, x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps): fn(h, x.data_ptr(), y.data_ptr())
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / reps)
    return outs, times
for n in (128, 256, 512, 1024):
    a, ta = run(0, n, 10 if n == 1024 else 20)
    b, tb = run(1, n, 10 if n == 1024 else 20)
    print(n, "bitwise", [np.array_equal(u, v) for u, v in zip(a, b)], "cluster ms", ["%.4f" % t for t in ta],
          "decoupled ms", ["%.4f" % t for t in tb], flush=True)
