"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys


def main(path, steps=1, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = re.sub(r"\(.*", "", r[ki])[:100]
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"launches {sum(cnt.values())}  total {allt/1e6:.3f} ms")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        print(f"{v/1e6/steps:9.3f} ms/step {100*v/allt:5.1f}%  n={cnt[k]//steps:5d}/step  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
