"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0][:70]
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1000:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1000:9.3f} ms {100 * t / tot:5.1f}%  n={n:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
