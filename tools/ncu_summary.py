#!/usr/bin/env python
"""Summarise ncu captures into committed evidence under profiles/.

    python tools/ncu_summary.py --round r01 [gpurun_out/prof_G1.ncu-rep ...]

Writes profiles/<round>_ncu_summary.md (one row per capture: duration, DRAM
bytes read/written vs the algorithmic bytes, DRAM throughput, SM activity
spread, registers, occupancy), profiles/<round>_ncu_raw_<cfg>.csv (the key
raw metrics) and profiles/ncu_traffic.json (DRAM bytes per launch per config,
read by bench.py for the roofline `traffic` field).  Also summarises a
launch list (--launches gpurun_out/launches.csv) into
profiles/<round>_launches.md.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_active.avg", "sm__cycles_active.min", "sm__cycles_active.max",
    "sm__cycles_elapsed.max", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__inst_executed.sum", "launch__shared_mem_per_block_static",
]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def raw(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, h in enumerate(hdr):
        if h in KEYS or h == "Kernel Name":
            d[h] = (vals[i], units[i])
    return d


def num(d, k):
    v, u = d[k]
    x = float(v.replace(",", ""))
    return x * UNIT.get(u, 1.0)


def main():
    from paper_2108_02025_b200 import workloads as WL
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=None)
    ap.add_argument("reps", nargs="*")
    a = ap.parse_args()
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    traffic_path = prof / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    lines = [f"# ncu captures, round {a.round}", "",
             "`ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 1 -c 1` "
             "of `python tools/ncu_runner.py --config <cfg> --reps 2` on one B200 "
             "(ncu flushes caches before the replayed launch, so DRAM bytes are cold-cache). "
             "Algorithmic bytes: SURVEY.md §8(d).", "",
             "| cfg | kernel | grid x block | regs | duration us | DRAM read MB | DRAM write MB | "
             "alg MB | DRAM/alg | DRAM TB/s | SM active min/avg/max of elapsed |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for rep in a.reps:
        rep = Path(rep)
        cfg = rep.stem.split("_")[-1]
        d = raw(rep)
        dur = num(d, "gpu__time_duration.sum")
        rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
        if cfg == "R1x":  # GER fp32 8192 x 8193 (tools/ncu_runner.py)
            alg = (2 * 8192 * 8193 + 8192 + 8193) * 4
        elif cfg == "CM4096":  # col-major GEMV fp32 4096 x 16384
            alg = (4096 * 16384 + 16384 + 2 * 4096) * 4
        elif cfg == "RM1024":  # row-major GEMV fp32 65536 x 1024 (the sub-CTA sweep)
            alg = (65536 * 1024 + 1024 + 2 * 65536) * 4
        elif cfg == "RM1001":  # row-major GEMV fp32 67041 x 1001 (the scalar sub-CTA sweep)
            alg = (67041 * 1001 + 1001 + 2 * 67041) * 4
        else:  # D1f / G1g: D1 / G1 through the fused peer-memory paths
            alg = WL.WORKLOADS[cfg[:2]].alg_bytes(1)
        el = num(d, "sm__cycles_elapsed.max")
        act = [num(d, f"sm__cycles_active.{s}") / el for s in ("min", "avg", "max")]
        kname = d["Kernel Name"][0].split("(")[0].replace("void ", "")
        lines.append(f"| {cfg} | `{kname[:60]}` | {d['launch__grid_size'][0]} x "
                     f"{d['launch__block_size'][0]} | {d['launch__registers_per_thread'][0]} | "
                     f"{dur * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {alg / 1e6:.1f} | "
                     f"{(rd + wr) / alg:.3f} | {(rd + wr) / dur / 1e12:.2f} | "
                     f"{act[0]:.2f} / {act[1]:.2f} / {act[2]:.2f} |")
        with open(prof / f"{a.round}_ncu_raw_{cfg}.csv", "w") as f:
            f.write("metric,unit,value\n")
            for k, (v, u) in sorted(d.items()):
                f.write(f"{k},{u},\"{v}\"\n")
        traffic[cfg] = {"dram_bytes_per_launch": int(rd + wr), "alg_bytes": alg,
                        "ncu_duration_us": round(dur * 1e6, 3), "kernel": kname,
                        "source": f"profiles/{a.round}_ncu_raw_{cfg}.csv (ncu --set full)"}
    if a.reps:
        (prof / f"{a.round}_ncu_summary.md").write_text("\n".join(lines) + "\n")
        traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = collections.OrderedDict()
        for r in rows[1:]:
            agg.setdefault(r[ki].split("(")[0].replace("void ", "")[:90], []).append(
                float(r[vi].replace(",", "")))
        total = sum(sum(v) for v in agg.values())
        out = [f"# launch list, round {a.round}", "",
               "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` of "
               "`python bench.py --steps 20 --warmup 3 --no-suite --no-e2e --no-cpu-baseline` "
               "(cold-cache, serialised: compare shares, not absolutes).  fill_* seed the inputs; "
               "the at:: kernels are the L2 flush (write + read of 512 MiB) that bench.py runs "
               "before timing / between flushed steps; cuda::spin_kernel is torch.cuda._sleep, the "
               "0.5 ms device sleep the timed steps queue behind (before the start event).  "
               "G1 steps run back to back (inputs 2.1x "
               f"the L2, see {a.round}_ncu_b2b_G1.csv), so the step is one launch of the GEMV kernel.",
               "",
               "| kernel | launches | mean us | share of all GPU time |", "|---|---|---|---|"]
        for k, v in agg.items():
            out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / total:.3f} |")
        (prof / f"{a.round}_launches.md").write_text("\n".join(out) + "\n")
        import shutil
        shutil.copy(a.launches, prof / f"{a.round}_launches.csv")


if __name__ == "__main__":
    main()
