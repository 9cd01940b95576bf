"""Summarize an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) per kernel name:
launches, device time, share of the step, DRAM bytes.
    python tools/launch_summary.py gpurun_out/launches.csv [profiles/traffic.json]"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik, im, iu, iv = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    launches = collections.defaultdict(set)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
             "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        val = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
        per[name][r[im]] += val
        launches[name].add(r[0])
    total_t = sum(d["gpu__time_duration.sum"] for d in per.values())
    print(f"{'kernel':70s} {'n':>5} {'ms':>8} {'share':>6} {'DRAM MB':>9} {'GB/s':>7}")
    for name, d in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = d["gpu__time_duration.sum"]
        b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        print(f"{name[:70]:70s} {len(launches[name]):>5} {t*1e3:>8.3f} {t/total_t:>6.1%} "
              f"{b/1e6:>9.1f} {b/t/1e9 if t else 0:>7.0f}")
    print(f"total {total_t*1e3:.3f} ms (serialised, cold-cache launches)")
    if len(sys.argv) > 2:
        # DRAM traffic per step of the per-layer kernel classes bench.py reports
        cls = {"fwd_layer_kernel": 0.0, "bwd_layer_kernel": 0.0}
        for name, d in per.items():
            b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            if name.startswith(("items_kernel", "combine_kernel")):
                cls["bwd_layer_kernel" if "BwdGather" in name else "fwd_layer_kernel"] += b
        import json
        with open(sys.argv[2], "w") as fh:
            json.dump({"source": path, "unit": "bytes per step", **cls}, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
