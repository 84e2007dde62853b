"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, out_path, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else v * 1000 if r[ui] == "ms" else v
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    with open(out_path, "w") as f:
        f.write(title + "\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f"{k:44s} launches={cnt[k]:5d} total_us={tot[k]:10.1f} share={tot[k] / T * 100:5.1f}% "
                    f"avg_us={tot[k] / cnt[k]:8.2f}\n")
    print(open(out_path).read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
