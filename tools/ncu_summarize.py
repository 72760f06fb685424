"""Summarise an `ncu --page source --csv` export: per kernel, total warp
stall samples by reason and the hottest SASS instructions.

    python tools/ncu_summarize.py gpurun_out/prof_source.csv.gz [top]
"""

import csv
import gzip
import io
import sys
from collections import defaultdict


def blocks(path):
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as f:
        text = f.read()
    cur_name, lines = None, []
    for line in text.splitlines():
        if line.startswith('"Kernel Name"'):
            if cur_name is not None:
                yield cur_name, lines
            cur_name = line.split(",", 1)[1].strip().strip(",").strip('"')
            lines = []
        else:
            lines.append(line)
    if cur_name is not None:
        yield cur_name, lines


def main(path, top=25):
    for name, lines in blocks(path):
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        if not rows:
            continue
        hdr = rows[0]
        idx = {h: i for i, h in enumerate(hdr)}
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        tot = defaultdict(float)
        insts = []
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            try:
                s = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
            except ValueError:
                continue
            for c in stall_cols:
                try:
                    tot[c] += float(r[idx[c]] or 0)
                except ValueError:
                    pass
            insts.append((s, r[idx["Address"]], r[idx["Source"]]))
        allsamp = sum(tot.values()) or 1
        print(f"==== {name}  (samples {allsamp:.0f})")
        for c, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
            print(f"   {c:28s} {100 * v / allsamp:5.1f}%")
        insts.sort(reverse=True)
        for s, a, src in insts[:top]:
            print(f"   {s:8.0f}  {a}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
