"""Static SASS instruction counts of the hot kernels in the built library
(cuobjdump -sass): the evidence for TMA (UTMALDG / UTMASTG / UBLKCP),
async copies (LDGSTS), global / shared traffic and FP64 work per kernel.

    python profiles/sass_counts.py > profiles/r02/sass_counts.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2404_02433_b200" / "libetc_b200.so"
HOT = ["k_stencil_pht<512, 1, ", "k_stencil_gt<512, 1, ", "k_stencil_cp<512, 1, 1>",
       "k_fwd_q<512, 2, ", "k_inv_q<512, 1, 2, ", "k_zsolve_tma<16, ", "k_thomas_x<16, 8>", "k_fwd_c2<512, 2>",
       "k_inv_c2<512, 1, 2>", "k_zsub_ends", "k_zsub_solve", "k_op_stencil<double", "k_op_thomas<double",
       "k_op_ssor"]
OPS_F32 = ["FFMA", "FADD", "FMUL"]
OPS = ["UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "LDGSTS", "LDG", "STG", "LDS", "STS", "LDL", "STL", "DFMA",
       "DADD", "DMUL", "FFMA", "FADD", "FMUL", "MUFU", "SHFL", "BAR", "SYNCS", "RED", "ATOM", "UCGABAR"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    names = [re.sub(r"\((int|bool)\)", "", n) for n in re.findall(r"Function : ([^\n]+)", sass)]
    names = [subprocess.run(["cu++filt", n], capture_output=True, text=True).stdout.strip() if n.startswith("_Z")
             else n for n in names]
    names = [re.sub(r"\((int|bool)\)", "", n) for n in names]
    parts = re.split(r"\n\s*Function : [^\n]+", sass)[1:]
    print("# static SASS counts per kernel (cuobjdump -sass of paper_2404_02433_b200/libetc_b200.so)")
    print("# kernel | " + " ".join(OPS))
    for name, body in zip(names, parts):
        if not any(h in name for h in HOT):
            continue
        c = Counter(m.split(".")[0] for m in re.findall(r"\b([A-Z][A-Z0-9_]+(?:\.[A-Z0-9_]+)*)\b", body))
        print(f"{name.split('(')[0].replace('void ', '')[:44]:<44} | " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))


if __name__ == "__main__":
    sys.exit(main())
