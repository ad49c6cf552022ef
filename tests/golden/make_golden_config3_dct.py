"""Third rounding of the config-3 FCT cases: the oracle with its cosine
transforms as dense matrix products (oracle.precond_matmul), i.e. no FFT.
The perturbed oracle (make_golden_config3_floor.py) shares pocketfft's
transform rounding with the reference and the plain oracle; this variant
does not, so it measures the spread an independent transform implementation
(like the device's radix-8 plane FFTs) is entitled to at contrast 1000.
CPU only; writes tests/golden/solves_config3_dct.json.

    python tests/golden/make_golden_config3_dct.py
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import etc_oracle as O  # noqa: E402

HERE = Path(__file__).resolve().parent
out = []
for c in json.loads((HERE / "solves_config3.json").read_text()):
    if c["precond"] != "fct":
        continue
    n = c["n"]
    if c["kind"] == "fibres":
        fd = c["field"]
        kx = ky = kz = O.fibres(n, fd["count"], fd["r_min"], fd["r_max"], fd["kappa_fib"], fd["seed"], fd["axis"])
    else:
        kx, ky, kz = O.channels(8, n // 8, 3.0)
    t0 = time.time()
    r = O.homogenize(kx, ky, kz, (n, n, n, 1.0, 1.0, 1.0), c["axis"], 1.0, 0.0, c["rtol"], dct="matmul")
    out.append(dict(kind=c["kind"], n=n, axis=c["axis"], precond="fct", rtol=c["rtol"], iterations=r["iterations"],
                    kappa_eff=r["kappa_eff"], history=r["history"]))
    print(c["kind"], n, c["axis"], r["iterations"], c["iterations"],
          f"{abs(r['kappa_eff'] - c['kappa_eff']) / c['kappa_eff']:.2e}", f"{time.time() - t0:.0f}s", flush=True)
    (HERE / "solves_config3_dct.json").write_text(json.dumps(out) + "\n")
