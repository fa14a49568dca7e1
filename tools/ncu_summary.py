"""Summarise ncu output into profiles/ (run in the build container).

    python tools/ncu_summary.py launches <launches.csv> <out.json>
    python tools/ncu_summary.py full <report.ncu-rep> <out.json>

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel (cold-cache, serialised: compare shares, not absolutes).  `full`
extracts, per captured kernel, the duration, DRAM bytes, pipe utilisation,
occupancy and warp-stall breakdown of an `ncu --set full` capture.
"""

import collections
import csv
import io
import json
import subprocess
import sys


def _to_us(value, unit):
    v = float(value.replace(",", ""))
    return {"nsecond": v / 1e3, "usecond": v, "msecond": v * 1e3, "second": v * 1e6,
            "ns": v / 1e3, "us": v, "ms": v * 1e3, "s": v * 1e6}.get(unit, v)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        per[d["Kernel Name"].split("(")[0]].append(_to_us(d["Metric Value"], d["Metric Unit"]))
    total = sum(sum(v) for v in per.values())
    summary = sorted(({"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v),
                       "total_us": sum(v), "share": sum(v) / total} for k, v in per.items()),
                     key=lambda x: -x["total_us"])
    json.dump({"source": path, "total_us": total, "kernels": summary}, open(out, "w"), indent=1)
    for s in summary[:15]:
        print(f"{s['share'] * 100:5.1f}%  {s['mean_us']:9.1f} us x{s['launches']:3d}  {s['kernel']}")


WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "fp64_dadd",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "fp64_dmul",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "fp64_dfma",
    "smsp__inst_executed_pipe_fp64.sum": "fp64_warp_instructions",
}


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
             "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")[:80]}
        for m, name in WANT.items():
            if m in d and d[m] not in ("", "n/a"):
                try:
                    k[name] = float(d[m].replace(",", "")) * scale.get(units.get(m, ""), 1.0)
                except ValueError:
                    k[name] = d[m]
        stalls = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", ""))
                  for m, v in d.items()
                  if m.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not m.endswith("not_issued") and v not in ("", "0")}
        k["stall_samples"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
        if "dram_read_bytes" in k:
            k["dram_bytes"] = k["dram_read_bytes"] + k.get("dram_write_bytes", 0.0)
        if "fp64_dadd" in k:
            k["fp64_flops"] = (k.get("fp64_dadd", 0.0) + k.get("fp64_dmul", 0.0)
                               + 2.0 * k.get("fp64_dfma", 0.0))
            if k.get("duration_ns"):
                k["fp64_tflops"] = k["fp64_flops"] / k["duration_ns"] / 1e3
        kernels.append(k)
    json.dump({"source": path, "kernels": kernels}, open(out, "w"), indent=1)
    for k in kernels:
        print(json.dumps({x: k.get(x) for x in ("kernel", "duration_ns", "dram_bytes",
                                                  "fp64_pipe_pct", "occupancy_pct")}))


def step(path, out, steps="1"):
    """Whole-step DRAM traffic: a launch list captured with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
    over the last `steps` timed steps (cold-cache, serialised): per-kernel
    and total bytes per step."""
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0,
             "usecond": 1e3, "msecond": 1e6}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0]
        per[k][d["Metric Name"]] += float(d["Metric Value"].replace(",", "")) * scale.get(
            d["Metric Unit"], 1.0)
        ids[k].add(d["ID"])
    n = float(steps)
    kern = sorted(({"kernel": k, "launches_per_step": len(ids[k]) / n,
                    "dram_bytes_per_step": (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / n,
                    "ns_per_step": v["gpu__time_duration.sum"] / n} for k, v in per.items()),
                  key=lambda x: -x["dram_bytes_per_step"])
    total = sum(x["dram_bytes_per_step"] for x in kern)
    json.dump({"source": path, "steps": n, "dram_bytes_per_step": total, "kernels": kern},
              open(out, "w"), indent=1)
    print(f"DRAM bytes per step: {total / 1e6:.1f} MB")
    for x in kern[:12]:
        print(f"{x['dram_bytes_per_step'] / 1e6:8.2f} MB  {x['ns_per_step'] / 1e3:8.1f} us  {x['kernel']}")


if __name__ == "__main__":
    {"launches": launches, "full": full, "step": step}[sys.argv[1]](*sys.argv[2:])
