"""One-screen summary of an ncu --set full report: duration, issue activity,
pipe utilisation, DRAM bytes and the top stall reasons per kernel."""
import csv
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        d = dict(zip(h, v))
        f = lambda k: d.get(k, "?")  # noqa: E731
        print(d["Kernel Name"][:60], "| us", float(f("gpu__time_duration.sum")) / 1000 if "usecond" not in rows[1][h.index("gpu__time_duration.sum")] else f("gpu__time_duration.sum"))
        print("  issue%", f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "| warps/sched", f("smsp__warps_active.avg.per_cycle_active"),
              "| dram MB r/w", f("dram__bytes_read.sum"), f("dram__bytes_write.sum"),
              "| inst", f("smsp__inst_executed.sum"))
        pipes = []
        for k in h:
            if k.startswith("sm__inst_executed_pipe_") and k.endswith(".avg.pct_of_peak_sustained_active"):
                try:
                    x = float(d[k])
                except ValueError:
                    continue
                if x > 5:
                    pipes.append((x, k.replace("sm__inst_executed_pipe_", "").replace(".avg.pct_of_peak_sustained_active", "")))
        print("  pipes", ", ".join(f"{n} {x:.0f}%" for x, n in sorted(pipes, reverse=True)))
        for k in h:
            if "tensor" in k and "pct_of_peak_sustained_active" in k and k.startswith("sm__pipe"):
                print("  ", k, d[k])
        st = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1
        print("  stalls", ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
