"""Per-instruction stall profile from `ncu --page source --csv --print-source sass`:
prints the hottest SASS lines (by warp-stall samples) with their top stall reasons."""
import csv
import sys


def main(path, top=40, window=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    scols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # first kernel only
        if len(r) > wi and r[wi].isdigit():
            data.append(r)
    tot = sum(int(r[wi] or 0) for r in data)
    print(f"total samples {tot}")
    agg = {}
    for r in data:
        for i, h in scols:
            agg[h] = agg.get(h, 0) + int(r[i] or 0)
    print("  ".join(f"{h[6:]}={v / tot:.2f}" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for idx, r in enumerate(data):
        n = int(r[wi] or 0)
        if n < tot * 0.004:
            continue
        reasons = sorted(((int(r[i] or 0), h[6:]) for i, h in scols), reverse=True)[:3]
        rs = " ".join(f"{h}:{v}" for v, h in reasons if v)
        print(f"{idx:5d} {n:6d} {r[ei]:>9} {r[si].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1])
