"""Summarise ncu output (launch list CSV + a --set full report) into profiles/.

  python scripts/summarize_ncu.py <launches.csv> <full.ncu-rep[,more.ncu-rep]> <tag>

Writes profiles/<tag>_launches.md (per-kernel share of device time from the
serialized, cold-cache launch list), profiles/<tag>_gemm_full.md (per-launch DRAM
traffic / tensor-pipe utilisation / duration of the captured GEMM launches) and
profiles/ncu_traffic.json (mean DRAM bytes per GEMM launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("p2r::", "")
    return name[:70]


def launches(path):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        k = short(r["Kernel Name"])
        per[k][0] += 1
        per[k][1] += ns
    return per


def full_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[0], rows[2:]
    idx = {n: i for i, n in enumerate(hdr)}
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "lts__t_bytes.sum"]
    res = []
    for r in data:
        d = {"kernel": short(r[idx["Kernel Name"]])}
        for w in want:
            if w in idx:
                d[w] = r[idx[w]]
        res.append(d)
    units = {w: rows[1][idx[w]] for w in want if w in idx}
    return res, units


def to_bytes(v, unit):
    v = float(str(v).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    lpath, fpath, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    per = launches(lpath)
    tot = sum(v[1] for v in per.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             f"Source: `{os.environ.get('NCU_CMD', 'ncu --metrics gpu__time_duration.sum --clock-control none -c 700 python bench.py --steps 1 --warmup 1')}`",
             "(serialised, cold-cache per launch: compare SHARES with bench.py's live `kernels` breakdown, not absolutes).", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ns) in sorted(per.items(), key=lambda a: -a[1][1]):
        lines.append(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / tot:.3f} |")
    open(os.path.join(prof, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    res, units = [], {}
    for fp in fpath.split(","):
        r, u = full_report(fp)
        res += r
        units.update(u)
    lines = [f"# {tag}: ncu --set full on GEMM launches inside one bench step", "",
             "Captures: `ncu --set full --clock-control none -k regex:gemm_kernel --launch-skip 291 -c 4` (layer-0 forward:",
             "QKV, O-proj, FFN1, FFN2) and `--launch-skip 390 -c 10` (head + last-layer backward GEMMs) of",
             "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline`.", "",
             "| # | kernel | grid | duration | DRAM read | DRAM write | tensor pipe % of peak |", "|---|---|---|---|---|---|---|"]
    traffic = []
    for i, d in enumerate(res):
        rb = to_bytes(d.get("dram__bytes_read.sum", 0), units.get("dram__bytes_read.sum", "byte"))
        wb = to_bytes(d.get("dram__bytes_write.sum", 0), units.get("dram__bytes_write.sum", "byte"))
        traffic.append(rb + wb)
        lines.append(f"| {i} | `{d['kernel']}` | {d.get('launch__grid_size')} | "
                     f"{d.get('gpu__time_duration.sum')} {units.get('gpu__time_duration.sum', '')} | "
                     f"{rb / 1e6:.1f} MB | {wb / 1e6:.1f} MB | "
                     f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')} |")
    open(os.path.join(prof, f"{tag}_gemm_full.md"), "w").write("\n".join(lines) + "\n")
    if traffic:
        json.dump({"gemm": sum(traffic) / len(traffic), "_note": f"mean DRAM bytes per GEMM launch over {len(traffic)} "
                   f"launches of one C2 step ({tag}, ncu --set full)"},
                  open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
