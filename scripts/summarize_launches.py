"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import re
import sys


def short(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = re.sub(r"\(.*\)$", "", name)
    return name.replace("sqv::", "")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = short(r[iK])
        tot[k] += float(r[iV].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    # the bench's roofline denominators (mb_*: live SFU/FFMA peak
    # microbenchmarks) run once outside the timed steps: shares of the step
    # are over the remaining kernels
    Ts = sum(v for k, v in tot.items() if not k.startswith("mb_"))
    print(f"{'kernel':46s} {'launches':>8s} {'total us':>11s} {'share':>7s} {'of step':>8s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        step = "" if k.startswith("mb_") else f"{100 * v / Ts:7.1f}%"
        print(f"{k:46s} {cnt[k]:8d} {v / 1e3:11.1f} {100 * v / T:6.1f}% {step:>8s}")


if __name__ == "__main__":
    main(sys.argv[1])
