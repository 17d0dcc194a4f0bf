"""Turn ncu outputs into the summaries kept under profiles/ (measurement tool).

  python tools/ncu_summary.py --rep gpurun_out/prof_attn.ncu-rep --launches gpurun_out/launches.csv \
      --tag r01 --workload hunyuan720p

writes
  profiles/<tag>_ncu_full_summary.json   selected metrics of the --set full capture (tensor / XU / FMA / ALU pipes,
                                         DRAM bytes, L2 hit rate, warp-stall breakdown, top source lines)
  profiles/<tag>_launches_<workload>.csv per-kernel launch count, time, share of the step, DRAM bytes
  profiles/traffic_<workload>.json       DRAM bytes per attention launch (bench.py's roofline.traffic)
"""
import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def raw_metrics(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def source_hotspots(rep, top=15):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f, agg, total = None, [], 0
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "File Path":
            f = row[1].split("/")[-1]
        elif row and row[0].isdigit():
            try:
                n = int(row[4])
            except (ValueError, IndexError):
                continue
            agg.append((n, f"{f}:{row[0]}", row[1].strip()[:100]))
            total += n
    agg.sort(reverse=True)
    return [{"share": n / total, "line": loc, "source": src} for n, loc, src in agg[:top]] if total else []


def stall_breakdown(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in rows[2:]:
        for i in cols:
            try:
                tot[hdr[i]] += int(r[i] or 0)
            except ValueError:
                pass
    s = sum(tot.values())
    return {k: v / s for k, v in tot.most_common(8)} if s else {}


def launches(path):
    lines = open(path).read().splitlines()
    start = [k for k, ln in enumerate(lines) if ln.startswith('"ID"')][0]
    by = collections.defaultdict(dict)
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        d = by[int(r["ID"])]
        d["name"] = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("svg2::<unnamed>::", "")
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    agg = collections.OrderedDict()
    for _, d in sorted(by.items()):
        a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0)
        a[3] += d.get("dram__bytes_write.sum", 0.0)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--workload", default="hunyuan720p")
    args = ap.parse_args()
    m = raw_metrics(args.rep)
    summary = {"kernel": m.get("Kernel Name", ("", ""))[1],
               "metrics": {k: f"{m[k][1]} {m[k][0]}".strip() for k in KEYS if k in m},
               "stall_breakdown": stall_breakdown(args.rep), "source_hotspots": source_hotspots(args.rep)}
    os.makedirs("profiles", exist_ok=True)
    json.dump(summary, open(f"profiles/{args.tag}_ncu_full_summary.json", "w"), indent=1)
    rd = float(m["dram__bytes_read.sum"][1]) * UNIT[m["dram__bytes_read.sum"][0]]
    wr = float(m["dram__bytes_write.sum"][1]) * UNIT[m["dram__bytes_write.sum"][0]]
    json.dump({"kernel": summary["kernel"], "dram_bytes_per_launch": rd + wr,
               "source": f"ncu --set full --clock-control none, bench.py --profile-once ({args.workload}), {args.tag}",
               "note": "algorithmic minimum = Q+K+V read once + O written; the rest are K/V re-reads missing L2"},
              open(f"profiles/traffic_{args.workload}.json", "w"), indent=1)
    agg = launches(args.launches)
    tot = sum(a[1] for a in agg.values())
    with open(f"profiles/{args.tag}_launches_{args.workload}.csv", "w") as f:
        f.write(f"# ncu launch list, bench.py --profile-once ({args.workload}: cold call then one warm call), "
                f"--clock-control none; {sum(a[0] for a in agg.values())} launches, {tot / 1e6:.3f} ms serialised\n")
        f.write("kernel,launches,ms,share_pct,dram_read_GB,dram_write_GB\n")
        for n, a in agg.items():
            f.write(f"{n},{a[0]},{a[1] / 1e6:.4f},{a[1] / tot * 100:.2f},{a[2] / 1e9:.4f},{a[3] / 1e9:.4f}\n")
    print(json.dumps(summary["metrics"], indent=1))
    print(json.dumps(summary["stall_breakdown"], indent=1))


if __name__ == "__main__":
    main()
