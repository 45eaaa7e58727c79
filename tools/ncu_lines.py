"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > cs.csv
    python tools/ncu_lines.py cs.csv [top]
"""

import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, cur_src = "", None, ""
    agg = defaultdict(lambda: [0, 0, ""])
    hdr = None
    total = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        if r[0]:   # a source line row
            cur_line, cur_src = r[0], r[1]
            continue
        # sass row belonging to cur_line: columns align with hdr
        try:
            samples = int(r[4]) if r[4] not in ("", "-") else 0
            execd = int(r[7]) if r[7] not in ("", "-") else 0
        except (ValueError, IndexError):
            continue
        key = (cur_file, cur_line)
        agg[key][0] += samples
        agg[key][1] += execd
        agg[key][2] = cur_src
        total += samples
    items = sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]
    print(f"total samples {total}")
    for (f, ln), (s, e, src) in items:
        print(f"{100.0 * s / max(total, 1):5.1f}%  {f}:{ln:>5}  inst={e:>9}  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
