"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/ncu_summarize.py --launches gpurun_out/launches_r1.csv \
        --full gpurun_out/asym_dominant_r1.ncu-rep --key attn_score/compress \
        --elements 134217728 --alg-bytes 339738624 --tag r1

Writes profiles/ncu_summary.json (per-kernel dram bytes / duration from the
full capture, consumed by bench.py's roofline.traffic) and
profiles/<tag>_launches.md (the launch list of one bench step: per-kernel
cold-cache device time and DRAM bytes, and each kernel's share of the step).
"""
import argparse
import csv
import json
import subprocess
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROF = ROOT / "profiles"

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
]


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    kern = OrderedDict()
    for r in rows:
        if len(r) > 5 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"])
            kern.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return kern


def read_full(path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h, units, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
             "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}
    res = {}
    for m in FULL_METRICS:
        if m in h:
            i = h.index(m)
            try:
                res[m] = float(v[i].replace(",", "")) * scale.get(units[i], 1)
            except ValueError:
                res[m] = v[i]
    res["kernel"] = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--key", default="attn_score/compress")
    ap.add_argument("--elements", type=int, default=131072 * 1024)
    ap.add_argument("--alg-bytes", type=int, default=339738624)
    ap.add_argument("--tag", default="r1")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    summary_path = PROF / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {"kernels": {}}
    if a.full:
        f = read_full(a.full)
        traffic = f["dram__bytes_read.sum"] + f["dram__bytes_write.sum"]   # bytes
        dur_us = f["gpu__time_duration.sum"] / 1e3                          # ns -> us
        entry = {
            "tag": a.tag, "kernel": f["kernel"], "capture": Path(a.full).name,
            "dram_bytes_per_launch": int(traffic), "algorithmic_bytes_per_launch": a.alg_bytes,
            "traffic_over_algorithmic": round(traffic / a.alg_bytes, 4),
            "duration_us_under_ncu": round(dur_us, 2),
            "dram_gbs_under_ncu": round(traffic / dur_us / 1e3, 1),
            "instructions_per_element": round(f["smsp__inst_executed.sum"] * 32 / a.elements, 2),
            "metrics (bytes, ns, %)": {k: f[k] for k in FULL_METRICS if k in f},
        }
        summary["kernels"][a.key] = entry
        summary_path.write_text(json.dumps(summary, indent=1) + "\n")
        print(json.dumps(entry, indent=1))
    if a.launches:
        kern = read_launches(a.launches)
        total = sum(m.get("gpu__time_duration.sum", 0) for m in kern.values())
        lines = [f"# ncu launch list, one bench step ({a.tag})", "",
                 "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none --profile-from-start off python tools/ncu_step.py` "
                 "(cold-cache, serialised: compare shares, not absolutes).", "",
                 "| # | kernel | us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
        for (i, name), m in kern.items():
            t = m.get("gpu__time_duration.sum", 0)
            lines.append(f"| {i} | `{name.split('(')[0][:70]}` | {t / 1e3:.1f} | {t / total:.1%} | "
                         f"{m.get('dram__bytes_read.sum', 0) / 1e6:.2f} | {m.get('dram__bytes_write.sum', 0) / 1e6:.2f} |")
        lines += ["", f"Total kernel time {total / 1e3:.1f} us over {len(kern)} launches."]
        (PROF / f"{a.tag}_launches.md").write_text("\n".join(lines) + "\n")
        print("\n".join(lines[-3:]))


if __name__ == "__main__":
    main()
