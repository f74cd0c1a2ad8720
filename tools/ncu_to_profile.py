"""Summarise ncu reports / launch lists into profiles/ (run in the build container)."""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__shared_mem_per_block", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def report(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    x = float(v)
                    if m.startswith("dram__bytes"):
                        x *= UNIT.get(units[i], 1.0)
                        d[m] = x
                    elif m == "gpu__time_duration.sum":
                        d["time_us"] = x * {"ms": 1e3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}.get(units[i], 1.0)
                    else:
                        d[m] = x
                except ValueError:
                    d[m] = v
        if "dram__bytes_read.sum" in d:
            d["traffic_bytes"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= iv:
            continue
        try:
            x = float(r[iv].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        except ValueError:
            continue
        agg[r[ik].split("(")[0].replace("void ", "")].append(x)
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v), "last_us": v[-1]} for k, v in agg.items()}


if __name__ == "__main__":
    rnd, src, dst = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    summary = {"round": rnd, "reports": {}, "launch_lists": {}}
    for rep in sorted(src.glob(f"{rnd}_ncu_*.ncu-rep")):
        summary["reports"][rep.stem] = report(str(rep))
    for lst in sorted(src.glob(f"{rnd}_launches_*.csv")):
        summary["launch_lists"][lst.stem] = launches(str(lst))
    (dst / f"ncu_{rnd}.json").write_text(json.dumps(summary, indent=1))
    for name, ks in summary["reports"].items():
        for d in ks:
            print(f"{name:40s} {d['kernel'][:55]:55s} {d.get('time_us', 0):9.1f} us  traffic {d.get('traffic_bytes', 0)/1e6:9.1f} MB "
                  f"dram% {d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', '-')}  tensor% {d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', '-')}")
    for name, ks in summary["launch_lists"].items():
        print(name)
        for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["mean_us"] * kv[1]["launches"])[:8]:
            print(f"   {k[:60]:60s} n={v['launches']:3d} mean={v['mean_us']:9.1f} us last={v['last_us']:9.1f} us")
