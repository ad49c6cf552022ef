"""Top source lines by warp-stall samples from an ncu report's source page
(needs -lineinfo and --import-source on):  python profiles/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = sys.argv[3:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"] + (["-k", "regex:" + kf[0]] if kf else []),
                     capture_output=True, text=True).stdout
rows, path, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    if len(r) > 2 and r[2] != "-":
        continue  # SASS rows; the source rows carry the per-line totals
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    if s:
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                  and v.isdigit() and int(v) > 0}
        top3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        rows.append((s, path, int(r[0]), r[1].strip()[:70], top3))
tot = sum(x[0] for x in rows)
for s, p, ln, src, t3 in sorted(rows, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}% {p}:{ln:<5} {src:<70} {t3}")
