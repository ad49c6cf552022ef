"""Per-kernel times of the z-solve stage on z-slab ranks, pencil vs spike
(virtual ranks on one GPU: the kernels are the production ones, the exchange
is device copies).  Usage: python profiles/probes/spike_probe.py [n] [P] [mode ...]"""
import ctypes as C
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2404_02433_b200 as P  # noqa: E402
from paper_2404_02433_b200 import dist  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2
f = P.gen_random_balls(n, 40, 0.05, 0.15, 100.0, 11)
cube = f.kx.reshape(n, n, n).contiguous()
grid = (n, n, n, 1.0, 1.0, 1.0)
names = ["stencil", "fwd", "zsolve-A", "zsolve", "inv", "?", "other", "?"]
for mode in (sys.argv[3:] or ["pencil", "spike"]):
    comms = dist.ThreadComm.make(R)
    out = [None] * R

    def worker(r):
        torch.cuda.set_device(0)
        k0, nzl = dist.slab_bounds(n, R, r)
        k = cube[k0:k0 + nzl].contiguous().reshape(-1)
        ops = dist.CudaSlabOps(n, n, n, k0, nzl, R, r, 1.0, 1.0, 1.0)
        ops.lib.etc_profile(ops._h, 1)
        rep = dist.slab_solve(ops, comms[r], k, k, k, grid, 1.0, 0.0, 1e-6, zsolve=mode)
        ms = (C.c_double * 8)()
        cnt = (C.c_longlong * 8)()
        ops.lib.etc_profile_read(ops._h, ms, cnt, 1)
        out[r] = (rep, list(ms), list(cnt))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(R)]
    [t.start() for t in th]
    [t.join() for t in th]
    rep, ms, cnt = out[0]
    print(mode, "iterations", rep.iterations, "kappa", repr(rep.kappa_eff))
    for c in range(8):
        if cnt[c]:
            print("   class %d: %d launches, %.4f ms avg, %.4f ms per iteration (rank 0)"
                  % (c, cnt[c], ms[c] / cnt[c], ms[c] / (rep.iterations + 1)))
