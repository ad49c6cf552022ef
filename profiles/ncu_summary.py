"""Summarise an `ncu --set full` capture (run here on the .ncu-rep brought
back from the GPU box) into the committed text summary and the per-kernel
DRAM traffic that bench.py reports as roofline.traffic.

    python profiles/ncu_summary.py gpurun_out/prof512h.ncu-rep profiles/r01/ncu_full_512
"""

import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "GB"),
    ("dram__bytes_write.sum", "GB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("launch__registers_per_thread", ""),
    ("launch__grid_size", ""),
    ("launch__cluster_dim_x", ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", ""),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
]
STALLS = ["long_scoreboard", "barrier", "short_scoreboard", "mio_throttle", "wait", "math_pipe_throttle",
          "lg_throttle", "not_selected", "membar", "dispatch_stall"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def num(v):
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


def main(rep, stem):
    hdr, units, rows = raw(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary of {rep} (one launch per kernel)"]
    traffic = {}
    for r in rows:
        name = r[ix["Kernel Name"]]
        lines.append("----")
        lines.append(f"  kernel: {name}")
        for m, _ in METRICS:
            if m in ix:
                lines.append(f"  {m}: {r[ix[m]]} {units[ix[m]]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in ix and num(r[ix[k]]) is not None:
                st.append((num(r[ix[k]]), s))
        st.sort(reverse=True)
        lines.append("  top stalls (warps per issue): " + " ".join(f"{s}={v:.2f}" for v, s in st[:6]))
        rd, wr = num(r[ix["dram__bytes_read.sum"]]), num(r[ix["dram__bytes_write.sum"]])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[ix["dram__bytes_read.sum"]]]
        scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[ix["dram__bytes_write.sum"]]]
        short = name.split("(")[0].replace("void ", "").strip()
        traffic[short] = {"dram_bytes": rd * scale + wr * scale_w,
                          "ms": num(r[ix["gpu__time_duration.sum"]])}
    open(stem + "_summary.txt", "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(stem + "_traffic.json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
