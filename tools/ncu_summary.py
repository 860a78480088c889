"""Summarise an ncu report (or a launch-list CSV) into a small JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_c2.json [--label ...]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/launches_c2.json
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed.sum": "warp_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "smsp__inst_executed_op_shared_ld.sum": "lds",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def summarise(rep, label):
    kernels = []
    for hdr, units, row in raw(rep):
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "")[:160], "label": label}
        for src, dst in KEYS.items():
            if src in d and d[src] not in ("", "n/a"):
                try:
                    v = float(d[src].replace(",", ""))
                except ValueError:
                    continue
                unit = u.get(src, "")
                if dst in ("duration",):
                    v *= UNIT_SCALE.get(unit, 1e-9)
                elif dst.startswith("dram"):
                    v *= UNIT_SCALE.get(unit, 1)
                k[dst] = v
        stalls = {h.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(d[h]) for h in hdr
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and d[h] not in ("", "n/a")
                  and not h.endswith("_not_issued")}
        tot = sum(stalls.values()) or 1.0
        k["stall_share_top"] = dict(sorted(((s, round(v / tot, 3)) for s, v in stalls.items()),
                                           key=lambda x: -x[1])[:6])
        if "dram_read" in k:
            k["dram_bytes_per_launch"] = k.get("dram_read", 0) + k.get("dram_write", 0)
        kernels.append(k)
    return kernels


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        out.append({"kernel": d["Kernel Name"][:120], "ns": v * (1 if d["Metric Unit"] == "ns" else
                                                              1e3 if d["Metric Unit"] == "us" else 1e6)})
    total = sum(x["ns"] for x in out) or 1.0
    for x in out:
        x["share"] = round(x["ns"] / total, 4)
    return {"launches": out, "total_ns": total}


def main():
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        res = launches(args[1])
        dst = args[2]
    else:
        label = ""
        if "--label" in args:
            i = args.index("--label")
            label = args[i + 1]
            del args[i:i + 2]
        res = summarise(args[0], label)
        dst = args[1]
        if len(res) == 1:
            res = res[0]
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
