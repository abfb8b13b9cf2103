"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): the last
``--tail`` launches, per kernel name, with durations in microseconds."""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tail", type=int, default=8)
    args = ap.parse_args()
    hdr, data = None, []
    for r in csv.reader(open(args.csv)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot = 0.0
    for d in data[-args.tail:]:
        us = float(d["Metric Value"]) / 1e3
        tot += us
        print(f"{us:10.1f} us  grid {d.get('Grid Size', ''):>14}  {d['Kernel Name'][:80]}")
    print(f"{tot:10.1f} us  total of the last {args.tail} launches")


if __name__ == "__main__":
    main()
