"""Fused float32 solve (ETC_FAST32=1, default) against the plain float32
kernels (ETC_FAST32=0) and the float64 solve: iterations, kappa_eff,
history agreement and device time per iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def solve(f, ax, prec, fast, rtol=1e-6):
    os.environ["ETC_FAST32"] = str(fast)
    P.release_plans()
    rep = P.homogenize(f, P.BoundaryConfig(P.Axis(ax), 1.0, 0.0), rtol, precision=prec)
    rep2 = P.homogenize(f, P.BoundaryConfig(P.Axis(ax), 1.0, 0.0), rtol, precision=prec)  # warm
    return rep2

cases = [("balls", 128, "z"), ("balls", 128, "x"), ("random", 128, "z"), ("balls", 256, "y"), ("balls", 512, "z"),
         ("random", 256, "x")]
for kind, n, ax in cases:
    if kind == "balls":
        f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
    else:
        g = P.GridSpec(n, n, n, 1.0, 1.0, 1.0)
        rng = np.random.default_rng(4)
        f = P.OrthotropicField(g, *np.exp(rng.uniform(-np.log(30), np.log(30), (3, n ** 3))))
    a = solve(f, ax, "f32", 1)
    b = solve(f, ax, "f32", 0)
    c = solve(f, ax, "f64", 1)
    m = min(len(a.relative_residuals), len(b.relative_residuals))
    ha, hb = np.array(a.relative_residuals[:m]), np.array(b.relative_residuals[:m])
    big = hb > 1e-2
    print(f"{kind} {n} {ax}: it fused {a.iterations} plain {b.iterations} f64 {c.iterations} | "
          f"kappa fused {a.kappa_eff:.9f} plain {b.kappa_eff:.9f} f64 {c.kappa_eff:.9f} | "
          f"rel fused-f64 {abs(a.kappa_eff-c.kappa_eff)/c.kappa_eff:.2e} plain-f64 {abs(b.kappa_eff-c.kappa_eff)/c.kappa_eff:.2e} | "
          f"hist dev {np.max(np.abs(ha[big]-hb[big])/hb[big]) if big.any() else 0:.2e} | "
          f"ms/it fused {a.device_ms/max(1,a.iterations):.3f} plain {b.device_ms/max(1,b.iterations):.3f} "
          f"f64 {c.device_ms/max(1,c.iterations):.3f}", flush=True)
