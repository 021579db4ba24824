"""Summarise `ncu --set full` reports of the attention kernels into a markdown table:
python scripts/summarize_attn_ncu.py out.md rep1.ncu-rep [rep2 ...]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %", 1),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2]))


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[1], rows[2:]
    cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(float(r[h.index("Warp Stall Sampling (All Samples)")] or 0) for r in data)
    agg = {h[i][6:]: sum(float(r[i] or 0) for r in data) / tot * 100 for i in cols}
    return sorted(agg.items(), key=lambda x: -x[1])[:4]


def main(out, reps):
    lines = ["# r01: attention kernels, `ncu --set full --clock-control none` (one launch each, "
             "`scripts/attn_bench.py`: B=8, H=16, S=1024, hd=64, causal)", "",
             "Per-launch metrics are cold-cache and serialised (ncu replay); compare with the live "
             "CUDA-event timings in DESIGN.md §3.1.", "",
             "| kernel | " + " | ".join(m[1] for m in METRICS) + " | top stall reasons (% of samples) |",
             "|---|" + "---|" * (len(METRICS) + 1)]
    for rep in reps:
        r = raw(rep)
        name = rep.split("/")[-1].replace(".ncu-rep", "").replace("r01_", "")
        vals = []
        for key, _, scale in METRICS:
            v = r.get(key)
            vals.append(f"{float(v) * scale:.1f}" if v not in (None, "") else "n/a")
        st = ", ".join(f"{k} {v:.0f}" for k, v in stalls(rep))
        lines.append(f"| `{name}` | " + " | ".join(vals) + f" | {st} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
