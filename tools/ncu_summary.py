"""Summarise an `ncu --set full` report into the JSON committed under profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json --what "..." [--algorithmic-bytes B ...]

Per launch: duration, DRAM read / write bytes (`traffic`), DRAM throughput,
FP64 pipe and issue activity, shared-memory wavefronts and bank conflicts,
registers, and the top warp-stall reasons (pc sampling).  `--algorithmic-
bytes` (one per launch, in order) adds the algorithmic traffic the bench
counts for that launch, so traffic / algorithmic shows re-reads.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
    "sm_cycles": ("sm__cycles_elapsed.avg", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "s": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--what", default="")
    ap.add_argument("--algorithmic-bytes", type=float, nargs="*", default=[])
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    launches = []
    for li, d in enumerate(data):
        out = {"kernel": d[col["Kernel Name"]].split("(")[0]}
        for key, (name, scale) in METRICS.items():
            if name not in col:
                continue
            v, u = _num(d[col[name]]), units[col[name]]
            if key == "duration_ms":
                v = v * UNIT.get(u, 1.0) * 1e3
            elif key.endswith("_bytes"):
                v = v * UNIT.get(u, 1.0)
            out[key] = v
        out["traffic_bytes"] = out.get("dram_read_bytes", 0.0) + out.get("dram_write_bytes", 0.0)
        if li < len(a.algorithmic_bytes):
            out["algorithmic_bytes"] = a.algorithmic_bytes[li]
            out["traffic_over_algorithmic"] = out["traffic_bytes"] / a.algorithmic_bytes[li]
            out["achieved_gbs_under_ncu"] = a.algorithmic_bytes[li] / (out["duration_ms"] * 1e-3) / 1e9
        stalls = {}
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = _num(d[i])
        tot = sum(stalls.values()) or 1.0
        out["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        out["what"] = a.what
        launches.append(out)
    json.dump({"report": a.report, "command": a.command, "launches": launches}, open(a.out, "w"), indent=1)
    print(json.dumps(launches, indent=1)[:3000])


if __name__ == "__main__":
    main()
