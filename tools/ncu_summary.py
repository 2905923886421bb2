"""Summaries of ncu output for profiles/ (read here, never on the timed path).

    python tools/ncu_summary.py launches <launch-list.csv>      # per-kernel share of the step
    python tools/ncu_summary.py full <report.ncu-rep>           # key --set full counters

The launch list is the `--metrics gpu__time_duration.sum --clock-control none` pass
(per-launch, serialised, cold-cache: the SHARE is comparable with bench.py, not the
absolute time). The full summary keeps the counters DESIGN.md cites: tensor-pipe and XU
utilisation, DRAM bytes (the roofline `traffic`), duration and clocks."""
import collections
import csv
import io
import json
import subprocess
import sys

FULL_KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def _ns(v, unit):
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9}
    return float(v) * scale.get(unit, 1.0)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += _ns(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [{"kernel": k, "launches": n, "total_us": round(t / 1e3, 1), "share": round(t / tot, 4),
            "us_per_launch": round(t / n / 1e3, 2)} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    return {"source": path, "launches": len(data), "kernels": out}


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in FULL_KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = f"{r[i]} {units[i]}".strip()
        out.append(rec)
    return {"source": path, "kernels": out}


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
