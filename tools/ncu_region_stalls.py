"""Stall reasons per source region: joins the cuda,sass and sass source pages by address.

    ncu -i rep --page source --csv --print-source=cuda,sass > cs.csv
    ncu -i rep --page source --csv --print-source=sass > s.csv
    python tools/ncu_region_stalls.py cs.csv s.csv
"""
import csv
import sys
from collections import defaultdict

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_regions import REGIONS  # noqa: E402


def main():
    where = {}
    cur_file, cur_line, hdr = "", 0, None
    for r in csv.reader(open(sys.argv[1])):
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
        name = cur_file
        for f, lo, hi, nm in REGIONS:
            if f == cur_file and lo <= cur_line <= hi:
                name = nm
                break
        where[r[2]] = name
    hdr = None
    agg = defaultdict(lambda: defaultdict(int))
    for r in csv.reader(open(sys.argv[2])):
        if "Address" in r and "# Samples" in r:
            hdr = r
            idx = {h: i for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h}
            continue
        if hdr and len(r) == len(hdr):
            reg = where.get(r[0], "?")
            for h, i in idx.items():
                try:
                    agg[reg][h] += int(r[i] or 0)
                except ValueError:
                    pass
    tot = sum(sum(v.values()) for v in agg.values())
    print(f"{'region':30s} {'all%':>6s} {'nonbar%':>7s}  top non-barrier reasons")
    for reg, v in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(v.values())
        nb = s - v.get("stall_barrier", 0)
        top = sorted(((c, h) for h, c in v.items() if h != "stall_barrier"), reverse=True)[:3]
        print(f"{reg:30s} {100 * s / tot:6.1f} {100 * nb / tot:7.1f}  " +
              ", ".join(f"{h[6:]} {100 * c / tot:.1f}" for c, h in top if c))


if __name__ == "__main__":
    main()
