"""Summarise ESP_GEMM_TRACE stamps (tools/skinny_probe.py run with
ESP_GEMM_TRACE=<file>): per launch, median/max over CTAs of the phases
relative to the earliest CTA entry, in microseconds."""
import statistics
import sys


def main(path):
    launches, cur = [], None
    for line in open(path):
        if line.startswith("launch"):
            cur = [line.strip(), []]
            launches.append(cur)
        else:
            v = [int(x) for x in line.split()[1:]]
            cur[1].append(v)
    names = ["entry", "setup", "first_stage", "mma_done", "epi_done", "exit", "first_drain"]
    seen = set()
    for hdr, rows in launches[-40:]:
        key = hdr.split(" per=")[0] + hdr.split(" grid=")[0][-8:]
        t0 = min(r[0] for r in rows)
        end = max(r[5] for r in rows)
        stats = []
        for i, n in enumerate(names):
            xs = [(r[i] - t0) / 1e3 for r in rows if r[i]]
            if xs:
                stats.append(f"{n} {statistics.median(xs):.1f}/{max(xs):.1f}")
        print(f"{hdr}: span {(end - t0) / 1e3:.1f} us | " + " | ".join(stats))


if __name__ == "__main__":
    main(sys.argv[1])
