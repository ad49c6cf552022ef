"""Bitwise fingerprint of the float64 kernels (plane transforms, z-solve,
preconditioner, stencils, whole solves): sha256 of each output.  Run before
and after a refactor that must not change float64 results; compare the JSON."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P

def h(t):
    return hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()[:16]

out = {}
for n in (64, 128, 256, 512):
    P.release_plans()
    g = P.GridSpec(n, n, n, 1.0, 1.0, 1.0)
    rng = np.random.default_rng(3)
    k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, n ** 3)))
    ds = P.DeviceSystem(P.OrthotropicField(g, *k))
    torch.manual_seed(1)
    x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    lib, hd = ds.plan.lib, ds.plan.handle
    for name in ("etc_dct2_xy", "etc_dct3_xy", "etc_apply_precond", "etc_apply_operator"):
        getattr(lib, name)(hd, x.data_ptr(), y.data_ptr()); torch.cuda.synchronize()
        out[f"{name}@{n}"] = h(y)
    z = x.clone(); lib.etc_thomas(hd, z.data_ptr()); torch.cuda.synchronize()
    out[f"etc_thomas@{n}"] = h(z)
    del ds
for n, ax in ((128, "x"), (256, "z"), (512, "y")):
    P.release_plans()
    f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
    rep = P.homogenize(f, P.BoundaryConfig(P.Axis(ax), 1.0, 0.0), 1e-6)
    out[f"solve-balls@{n}{ax}"] = [rep.iterations, repr(rep.kappa_eff),
                                   hashlib.sha256(np.array(rep.relative_residuals).tobytes()).hexdigest()[:16]]
P.release_plans()
g = P.GridSpec(128, 128, 128, 1.0, 1.0, 1.0)
rng = np.random.default_rng(4)
k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, 128 ** 3)))
rep = P.homogenize(P.OrthotropicField(g, *k), P.BoundaryConfig(P.Axis.X, 1.0, 0.0), 1e-8)
out["solve-random@128x"] = [rep.iterations, repr(rep.kappa_eff),
                            hashlib.sha256(np.array(rep.relative_residuals).tobytes()).hexdigest()[:16]]
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out))
