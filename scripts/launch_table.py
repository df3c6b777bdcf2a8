"""Summarise an ncu launch list (gpu__time_duration.sum CSV) into a per-kernel share table."""
import collections
import csv
import sys


def main(path, out, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
             "msecond": 1.0, "s": 1e3, "second": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[mi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(title + "\n\n| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f"| `{k}` | {cnt[k]} | {tot[k]:.3f} | {tot[k] / cnt[k]:.3f} | {tot[k] / T:.3f} |\n")
    print(open(out).read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
