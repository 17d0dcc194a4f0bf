"""Per-kernel roofline table from one ncu metrics pass over a whole bench call (measurement tool, not product):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,\
sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second \
      --clock-control none --csv --log-file every.csv python bench.py --profile-once
  python tools/ncu_every_kernel.py every.csv profiles/<tag>_every_kernel_<workload>.csv

For every kernel name: launches, mean time per launch, DRAM bytes per launch, achieved DRAM GB/s and its fraction of
the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs; the fallback of B200_PROFILING.md if absent), the tensor
pipe's active fraction and ncu's DRAM / SM throughput percentages (launch averages).  Per-launch times are
cold-cache and serialised (ncu), so compare shares and rates, not absolute call times."""
import collections
import csv
import io
import json
import os
import re
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    lines = open(src).read().splitlines()
    start = [k for k, ln in enumerate(lines) if ln.startswith('"ID"')][0]
    by = collections.defaultdict(dict)
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        d = by[int(r["ID"])]
        d["name"] = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("svg2::<unnamed>::", "")
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e6, "us": 1e3, "nsecond": 1.0,
                 "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
        peak_src = "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        peak, peak_src = 7700.0, "B200_PROFILING.md fallback"
    agg = collections.OrderedDict()
    for _, d in sorted(by.items()):
        if "svg2" not in d["name"] and not d["name"].startswith("k_"):
            continue  # torch's own helper kernels (allocator memsets, reductions in the bench harness)
        a = agg.setdefault(d["name"], collections.defaultdict(float))
        a["n"] += 1
        for k, v in d.items():
            if k != "name":
                a[k] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    with open(dst, "w") as f:
        f.write(f"# one ncu metrics pass over bench.py --profile-once (cold call, then one warm call), --clock-control "
                f"none; serialised launches; HBM peak {peak:.1f} GB/s ({peak_src})\n")
        f.write("kernel,launches,us_per_launch,share_pct,dram_MB_per_launch,dram_GBps,hbm_frac,tensor_pipe_pct,"
                "dram_throughput_pct,sm_throughput_pct,sm_ghz\n")
        for name, a in agg.items():
            n = a["n"]
            t = a["gpu__time_duration.sum"] / n  # ns
            by_ = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / n
            gbs = by_ / t if t else 0.0
            f.write(f"{name},{int(n)},{t / 1e3:.1f},{a['gpu__time_duration.sum'] / tot * 100:.2f},{by_ / 1e6:.1f},"
                    f"{gbs:.0f},{gbs / peak:.3f},"
                    f"{a['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'] / n:.1f},"
                    f"{a['dram__throughput.avg.pct_of_peak_sustained_elapsed'] / n:.1f},"
                    f"{a['sm__throughput.avg.pct_of_peak_sustained_elapsed'] / n:.1f},"
                    f"{a['sm__cycles_elapsed.avg.per_second'] / n / 1e9:.3f}\n")
    print(open(dst).read())


if __name__ == "__main__":
    main()
