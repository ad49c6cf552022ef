"""One 512^3 z-solve configuration for ncu (ETC_ZTMA selects the kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2404_02433_b200 as P
n = int(os.environ.get("ZN", "512"))
g = P.GridSpec(n, n, n, 1.0, 1.0, 1.0)
rng = np.random.default_rng(5)
k = np.exp(rng.uniform(-np.log(30), np.log(30), (3, n ** 3)))
ds = P.DeviceSystem(P.OrthotropicField(g, *k))
x = torch.from_numpy(rng.standard_normal(n ** 3)).cuda()
for _ in range(5):
    ds.plan.lib.etc_thomas(ds.plan.handle, x.data_ptr())
torch.cuda.synchronize()
print("ok")
