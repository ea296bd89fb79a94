"""Summarise an ncu --metrics gpu__time_duration.sum launch list: share per kernel."""
import collections
import csv
import sys


def summarise(path, skip_names=("k_gemm_s8", "k_build_enc", "k_build_dec")):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    out = ["total %.2f ms over %d launches" % (s / 1e6, sum(cnt.values()))]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
        out.append("%-44s %9.2f ms %5.1f%%  n=%5d  avg=%8.1f us" % (k, v / 1e6, 100 * v / s, cnt[k], v / cnt[k] / 1e3))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
