"""Top SASS instructions by warp-stall samples with their dominant stall reasons.

    ncu -i rep.ncu-rep --page source --csv --print-source=sass > /tmp/s.csv
    python tools/ncu_sass_stalls.py /tmp/s.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Address" in r and "# Samples" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    i_s = hdr.index("# Samples")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    src_i = hdr.index("Source")
    adr_i = hdr.index("Address")
    tot = sum(float(r[i_s] or 0) for r in data)
    data.sort(key=lambda r: -float(r[i_s] or 0))
    print(f"total samples {tot:.0f}")
    for r in data[:top]:
        n = float(r[i_s] or 0)
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        why = ", ".join(f"{k} {100 * v / max(n, 1):.0f}%" for v, k in st if v > 0)
        print(f"{100 * n / tot:5.1f}%  {r[adr_i]:>6}  {r[src_i][:60]:<60}  {why}")


if __name__ == "__main__":
    main()
