"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch) by kernel."""
import collections
import csv
import json
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        per[name][r[mi]] += v
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    return per, cnt


def main(path, out_json=None):
    per, cnt = load(path)
    tot = sum(m["gpu__time_duration.sum"] for m in per.values())
    print(f"| kernel | launches | share of time | avg us | DRAM read MB/launch | DRAM write MB/launch | GB/s |")
    print("|---|---|---|---|---|---|---|")
    res = {}
    for name, m in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = m["gpu__time_duration.sum"]
        n = cnt[name]
        rd, wr = m["dram__bytes_read.sum"] / n, m["dram__bytes_write.sum"] / n
        gbs = (rd + wr) / (t / n)  # bytes per ns = GB/s
        print(f"| {name} | {n} | {100*t/tot:.1f}% | {t/n/1e3:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {gbs:.0f} |")
        res[name] = {"launches": n, "share": t / tot, "avg_ns": t / n, "dram_bytes_per_launch": rd + wr}
    if out_json:
        json.dump(res, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
