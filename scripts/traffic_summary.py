"""Sum the ncu DRAM bytes of the kernels of ONE call per workload (scripts/traffic.sh).

usage: python scripts/traffic_summary.py <dir with traffic_<workload>.csv> <out.json>
Per workload: mean bytes read / written per launch of every kernel, then the per-call sum over the
kernels a call launches (each kernel name counted once per call)."""
import collections
import csv
import json
import os
import sys


def per_kernel(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "")
            unit, v = d.get("Metric Unit", ""), float(d["Metric Value"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                     "msecond": 1e6}.get(unit, 1)
            data[name][d["Metric Name"]].append(v * scale)
    return {k: {m: sum(v) / len(v) for m, v in mv.items()} | {"launches": len(mv["gpu__time_duration.sum"])}
            for k, mv in data.items()}


def main():
    src, out = sys.argv[1], sys.argv[2]
    res = {"_source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                      "--cache-control all --clock-control none over bench.py --workload <w> (scripts/traffic.sh); "
                      "per-launch means, per-call sum over the call's kernels"}
    for f in sorted(os.listdir(src)):
        if not (f.startswith("traffic_") and f.endswith(".csv")):
            continue
        w = f[len("traffic_"):-4]
        k = per_kernel(os.path.join(src, f))
        tot_r = sum(v.get("dram__bytes_read.sum", 0) for v in k.values())
        tot_w = sum(v.get("dram__bytes_write.sum", 0) for v in k.values())
        res[w] = {"kernels": k, "dram_bytes_read_per_call": tot_r, "dram_bytes_write_per_call": tot_w,
                  "dram_bytes_per_call": tot_r + tot_w}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    for w, v in res.items():
        if w.startswith("_"):
            continue
        print(w, {n: round(x.get("dram__bytes_read.sum", 0) / 1e6, 2) for n, x in v["kernels"].items()},
              "per call MB", round(v["dram_bytes_per_call"] / 1e6, 2))


if __name__ == "__main__":
    main()
