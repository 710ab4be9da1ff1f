"""Per-item phase timeline of tma_pass_kernel from a QV_TMA_TRACE build.

    QVB200_LIB=paper_2406_03466_b200/libqvb200_trace.so QVB200_TMA_TRACE=/tmp/t.bin \\
        QVB200_TMA_TRACE_LAUNCH=5 python tools/profile_pass.py 28 8 1
    python tools/tma_trace.py /tmp/t.bin

Prints, per team, the average SM cycles of each phase of an item (waiting
for the tile, each register group, the store + next-load issue) and the
item period, over the traced items of CTAs 0-3 (steady state: items 2..).
"""

import sys

import numpy as np


def main():
    raw = np.fromfile(sys.argv[1], dtype=np.int64)
    nm, ng, nstates, ntiles, blocks, teams, pieces, items = raw[:8]
    t = raw[8:].reshape(4, 2, items, 16)
    print(f"pass: {nm} matrices, {ng} groups; {nstates} states x {ntiles} tiles on {blocks} CTAs; "
          f"{teams} teams; {pieces} pieces")
    for team in range(int(teams)):
        rows = []
        for cta in range(4):
            for it in range(2, items - 1):
                e = t[cta, team, it]
                nxt = t[cta, team, it + 1]
                if e[0] == 0 or nxt[0] == 0:
                    continue
                r = {"wait": e[1] - e[0]}
                prev = e[1]
                for g in range(int(ng)):
                    r[f"g{g}"] = e[2 + g] - prev
                    prev = e[2 + g]
                if e[12]:   # the team's own thread stores and reloads the stage
                    r["tail"] = e[12] - prev      # last group's stores + fence + barrier
                    r["turn"] = e[13] - e[12]     # store issue, read-out wait, next load issue
                r["period"] = nxt[0] - e[0]
                rows.append(r)
        if not rows:
            continue
        keys = list(rows[0])
        avg = {k: float(np.mean([r[k] for r in rows])) for k in keys}
        print(f"team {team} ({len(rows)} items): " + ", ".join(f"{k} {v:.0f}" for k, v in avg.items()))


if __name__ == "__main__":
    main()
