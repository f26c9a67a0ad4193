"""Summarise ncu captures (.ncu-rep) and launch lists (.csv) for profiles/."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def rep(path, traffic=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")]
    print(f"kernel: {name}")
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k} = {vals[i]} {units[i]}")
    if traffic is not None:
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            tot += float(vals[i].replace(",", "")) * UNIT[units[i]]
        short = name.split("(")[0].split("::")[-1].split("<")[0]
        traffic[short] = tot


def launches(path):
    tot = defaultdict(lambda: [0.0, 0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.DictReader(io.StringIO("".join(lines)))
    for row in r:
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = row["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
        tot[k][0] += v
        tot[k][1] += 1
    s = sum(v[0] for v in tot.values())
    print(f"total device time {s / 1e3:.2f} ms over {sum(v[1] for v in tot.values())} launches")
    for k, (us, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"  {100 * us / s:6.2f}%  {us / 1e3:10.3f} ms  {n:5d} launches  {k}")


if __name__ == "__main__":
    # --traffic OUT.json: also write DRAM bytes per launch of each captured
    # kernel (read by bench.py for roofline.traffic).
    args = sys.argv[1:]
    out_json = None
    if args and args[0] == "--traffic":
        out_json, args = args[1], args[2:]
    traffic = {} if out_json else None
    for p in args:
        print(f"== {p}")
        if p.endswith(".csv"):
            launches(p)
        else:
            rep(p, traffic)
    if out_json:
        import json
        with open(out_json, "w") as f:
            json.dump(traffic, f, indent=1)
