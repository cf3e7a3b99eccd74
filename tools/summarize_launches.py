"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) into a markdown table
of kernel-class shares for profiles/.

  python tools/summarize_launches.py gpurun_out/launches.csv > profiles/roundN_launches.md
"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    names = {}
    for r in data:
        per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("vpe::", "").replace("<unnamed>::", "")
    return per, names


def main(path):
    per, names = load(path)
    tot, cnt, dram = collections.Counter(), collections.Counter(), collections.Counter()
    for i, m in per.items():
        n = names[i]
        tot[n] += m.get("gpu__time_duration.sum", 0.0)
        cnt[n] += 1
        dram[n] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    s = sum(tot.values())
    print(f"launches: {len(per)}; serialized sum of kernel durations: {s / 1e3:.1f} us\n")
    print("| kernel | launches | total us | share | DRAM MB |")
    print("|---|---:|---:|---:|---:|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / s:.1f}% | {dram[k] / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
