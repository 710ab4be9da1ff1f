"""Per-pass roofline breakdown from a QVB200_LAUNCH_LOG file.

    QVB200_LAUNCH_LOG=/tmp/l.txt python tools/one_gradient.py 28 8
    python tools/launch_breakdown.py /tmp/l.txt [--peak 6539.9]

Groups pass launches by kernel and matrices per pass; prints time, share,
algorithmic GB/s and fraction of the HBM peak (MEASURED_PEAKS.json) per
group, and the FP64 rate (28 flop counted per amplitude pair per matrix).
"""

import argparse
import collections
import json
from pathlib import Path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("log")
    ap.add_argument("--peak", type=float, default=None)
    ap.add_argument("--amp-bytes", type=int, default=16)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    peak = a.peak or json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    groups = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])   # launches, ms, bytes, flops
    for line in open(a.log):
        kern, m0, nm, ns, tiles, ms, by = line.split()
        nm, ns, tiles, ms, by = int(nm), int(ns), int(tiles), float(ms), float(by)
        amps = ns * tiles * 4096
        g = groups[(kern, nm)]
        g[0] += 1
        g[1] += ms
        g[2] += by
        g[3] += amps * 14.0 * nm
    total = sum(g[1] for g in groups.values())
    rows = []
    print(f"{'kernel':5s} {'mats':>4s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'GB/s':>8s} {'frac':>5s} {'TF/s':>6s}")
    for (kern, nm), (n, ms, by, fl) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        gbs = by / (ms * 1e-3) / 1e9 if ms else 0.0
        tfs = fl / (ms * 1e-3) / 1e12 if ms else 0.0
        rows.append({"kernel": kern, "matrices": nm, "launches": n, "ms": ms, "share": ms / total, "gbs": gbs,
                     "frac": gbs / peak, "fp64_tflops_counted": tfs})
        print(f"{kern:5s} {nm:4d} {n:8d} {ms:10.1f} {ms / total:6.3f} {gbs:8.0f} {gbs / peak:5.2f} {tfs:6.2f}")
    by_all = sum(g[2] for g in groups.values())
    print(f"all: {total:.1f} ms, {by_all / (total * 1e-3) / 1e9:.0f} GB/s = {by_all / (total * 1e-3) / 1e9 / peak:.3f} of {peak}")
    if a.json:
        json.dump({"peak_gbs": peak, "total_ms": total, "groups": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
