"""Executed-instruction and stall-sample totals per source region (file:line ranges).

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > cs.csv
    python tools/ncu_regions.py cs.csv
"""
import csv
import sys
from collections import defaultdict

REGIONS = [  # (file, lo, hi, name) -- first match wins
    ("hcs_greedy.cu", 170, 218, "solve: gather + fallback"),
    ("hcs_greedy.cu", 268, 273, "stop rule"),
    ("hcs_greedy.cu", 274, 302, "correlation"),
    ("hcs_greedy.cu", 303, 330, "select + union"),
    ("hcs_greedy.cu", 331, 375, "post-LS select"),
    ("hcs_greedy.cu", 376, 416, "residual"),
    ("hcs_greedy.cu", 417, 463, "cycle hash"),
    ("hcs_greedy.cu", 0, 10000, "greedy other"),
    ("hcs_ls_csne.cuh", 68, 98, "csne backward"),
    ("hcs_ls_csne.cuh", 100, 130, "csne forward"),
    ("hcs_ls_csne.cuh", 132, 145, "csne tile update"),
    ("hcs_ls_csne.cuh", 147, 215, "csne diag factor"),
    ("hcs_ls_csne.cuh", 226, 247, "csne gram"),
    ("hcs_ls_csne.cuh", 248, 300, "csne cholesky loop"),
    ("hcs_ls_csne.cuh", 301, 324, "csne guard+solve"),
    ("hcs_ls_csne.cuh", 325, 366, "csne refinement"),
    ("hcs_common.cuh", 0, 10000, "common (topk, reductions)"),
]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    cur_file, cur_line = "", 0
    agg = defaultdict(lambda: [0, 0])
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur_line = int(r[0])
            continue
        try:
            s = int(r[4]) if r[4] not in ("", "-") else 0
            e = int(r[7]) if r[7] not in ("", "-") else 0
        except (ValueError, IndexError):
            continue
        name = cur_file
        for f, lo, hi, nm in REGIONS:
            if f == cur_file and lo <= cur_line <= hi:
                name = nm
                break
        agg[name][0] += s
        agg[name][1] += e
    ts = sum(v[0] for v in agg.values())
    te = sum(v[1] for v in agg.values())
    print(f"{'region':32s} {'samples%':>8s} {'inst%':>7s}")
    for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:32s} {100 * s / ts:8.1f} {100 * e / te:7.1f}")


if __name__ == "__main__":
    main()
