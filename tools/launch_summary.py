"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel share of the LAST
forward (from the last forward_begin_kernel launch to the end)."""
import collections
import csv
import sys


def main(path, last_forward=True):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    dur, names = {}, {}
    for r in data:
        if r[mi] == "gpu__time_duration.sum":
            dur[int(r[idi])] = float(r[vi].replace(",", ""))
            names[int(r[idi])] = r[ki].split("(")[0].replace("void ", "").replace("dbl::", "")
    ids = sorted(dur)
    if last_forward:
        fb = [i for i in ids if "forward_begin" in names[i]]
        if fb:
            ids = [i for i in ids if i >= fb[-1]]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for i in ids:
        a = agg[names[i]]
        a[0] += 1
        a[1] += dur[i] / 1e3
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':58s} {'n':>5s} {'us':>10s} {'share':>7s}")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:58]:58s} {a[0]:5d} {a[1]:10.1f} {100 * a[1] / tot:6.1f}%")
    print(f"{'total':58s} {len(ids):5d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
