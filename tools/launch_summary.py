"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/launch_summary.py gpurun_out/launches_c2.csv
Prints per-kernel launches, total and average duration and share of the total.
ncu serialises launches and runs them cold-cache, so only the shares are
comparable with the bench's CUDA-event profile, not the absolute times.
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|unnamed>::", "", name)
    name = re.sub(r"\(CUtensorMap_st.*$|\(float \*.*$|\(int \*.*$|\(const .*$", "", name)
    return name.replace("void ", "").strip()


def main(path):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            r["Metric Unit"], 1e-3)
        tot[k] += v * scale
        cnt[k] += 1
    all_us = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {v / 1e3:10.2f} {v / cnt[k]:9.2f} {100 * v / all_us:6.1f}%")
    print(f"{'total':70s} {sum(cnt.values()):8d} {all_us / 1e3:10.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
