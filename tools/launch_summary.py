"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, total and
per-launch time and share of the listed GPU time, per kernel.

    python tools/launch_summary.py gpurun_out/launches_<tag>.csv [header line]
"""
import collections
import csv
import sys


def main(path, header=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                      hdr.index("Metric Value"))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    units = set()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        units.add(r[ui])
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    all_ms = sum(tot.values())
    if header:
        print(header)
    print(f"units seen: {sorted(units)}; cold-cache, serialised per-launch times; source: {path}")
    print(f"{'kernel':48s} {'launches':>8s} {'total_ms':>10s} {'ms/launch':>10s} {'share':>7s}")
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:48]:48s} {cnt[name]:8d} {t:10.3f} {t / cnt[name]:10.4f} {t / all_ms:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
