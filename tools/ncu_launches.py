"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"(k_\w+|Device\w+Kernel|\w+_kernel)", name)
    return m.group(1) if m else name[:40]


def main(path, out=None, last_steps=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit",
                                            "Metric Value"))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        a = agg.setdefault(short(r[ki]), [0.0, 0])
        a[0] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a[1] += 1
    tot = sum(a[0] for a in agg.values())
    lines = [f"# {sum(a[1] for a in agg.values())} launches, {tot / 1e3:.2f} ms of kernel time "
             "(ncu-serialised, cold cache; compare shares, not absolutes)",
             f"{'kernel':34s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}"]
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"{k:34s} {c:8d} {t / 1e3:10.3f} {t / c:10.2f} {100 * t / tot:6.2f}%")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
