"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total time and share of all listed time (the
launches are serialised and cold-cache under ncu, so compare shares, not
absolute times, with bench.py's live numbers).

    python tools/launch_summary.py gpurun_out/prof_launches.csv
"""
import collections
import csv
import re
import sys


def main(path):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 10 and r[0] != "ID"]
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[4]).replace("msk::<unnamed>::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[13], 1e-6)
        tot[name] += float(r[14].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {100 * v / all_ms:6.1f}%")
    print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_ms:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
