"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, mean duration and share of the total device time."""
import collections
import csv
import json
import sys


def summarise(path):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                rows.append(d)
    agg = collections.OrderedDict()
    for d in rows:
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "nsecond": 1e-6}.get(d["Metric Unit"], 1e-6)
        agg.setdefault(name, []).append(v * scale)
    total = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "mean_ms": sum(v) / len(v),
             "share": sum(v) / total} for k, v in agg.items()]


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1]), indent=1))
