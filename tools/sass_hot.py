"""Top SASS instructions by warp-stall samples from an ncu report's source page."""
import csv
import subprocess
import sys


def main(rep, n=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    body = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in body)
    print("total samples", tot, "instructions", len(body))
    idx = {r["Address"]: i for i, r in enumerate(body)}
    top = sorted(body, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:n]
    for r in top:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{idx[r['Address']]:5d} {100 * s / tot:5.1f}% {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
