"""Summarise a gpurun ncu capture into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/<tag> profiles/<round>_<workload> [--workload config0]

Reads <tag>/launches.csv (gpu__time_duration.sum per launch) and
<tag>/full.ncu-rep (--set full) and writes:
  <out>.md          per-kernel table: launches, mean device time, share of
                    the step, DRAM bytes, DRAM %, SM %, tensor-pipe %,
                    warps active, registers, top stall reasons
  <out>_launches.csv  the launch list (kernel, grid, block, ns)
and merges {workload: {kernel: dram bytes per launch}} into
profiles/ncu_traffic.json (bench.py reads `traffic` from it).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_rt_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem": "launch__shared_mem_per_block_dynamic",
    "inst": "smsp__inst_executed.sum",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, ig, ib = (hdr.index(x) for x in ("Kernel Name", "Metric Value", "Grid Size",
                                             "Block Size"))
    im = hdr.index("Metric Name") if "Metric Name" in hdr else None
    return [(short(r[ik]), r[ig], r[ib], float(r[iv].replace(",", ""))) for r in rows[1:]
            if (im is None or r[im] == "gpu__time_duration.sum") and "at::" not in r[ik]]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  or (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"))]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1) if k.startswith("dram_r") or k == "dram_wr" else v
        st = []
        for i in stall_cols:
            try:
                st.append((float(r[i].replace(",", "")), hdr[i].split("stalled_")[1]))
            except (ValueError, IndexError):
                pass
        d["stalls"] = [f"{n}" for v, n in sorted(st, reverse=True)[:4] if v > 0]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("out")
    ap.add_argument("--workload", default="config0")
    ap.add_argument("--title", default="")
    ap.add_argument("--launches", default="launches.csv", help="launch list file in <tag>")
    ap.add_argument("--full", default="full.ncu-rep", help="--set full report in <tag>")
    a = ap.parse_args()
    L = launches(os.path.join(a.tag, a.launches))
    with open(a.out + "_launches.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "block", "ns"])
        w.writerows(L)
    agg = collections.OrderedDict()
    for k, g, b, ns in L:
        agg.setdefault(k, []).append(ns)
    total = sum(ns for *_, ns in L)
    F = full(os.path.join(a.tag, a.full)) if os.path.exists(os.path.join(a.tag, a.full)) else []
    byk = collections.defaultdict(list)
    for d in F:
        byk[d["kernel"]].append(d)
    lines = [f"# {a.title or a.out}", "",
             f"Source: `{a.tag}` (ncu 2025, `--clock-control none`). Launch list = "
             "`--metrics gpu__time_duration.sum` over the whole command (cold, serialised); "
             "detail = `--set full` on the listed kernels.", "",
             "| kernel | launches | mean µs | share of launch time |", "|---|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | "
                     f"{sum(v) / total * 100:.1f} % |")
    lines += ["", "| kernel | µs | DRAM rd+wr B | DRAM % | SM % | tensor % | FMA % | warps % | "
              "regs | grid×block | inst | top stalls |", "|" + "---|" * 12]
    traffic = {}
    for k, ds in byk.items():
        for d in ds:
            tb = d.get("dram_rd", 0) + d.get("dram_wr", 0)
            traffic.setdefault(k, []).append(tb)
            lines.append(
                f"| `{k}` | {d.get('time_us', 0):.2f} | {tb:,.0f} | {d.get('dram_pct', 0):.2f} | "
                f"{d.get('sm_pct', 0):.1f} | {d.get('tensor_pct', d.get('tensor_rt_pct', 0)):.1f} | "
                f"{d.get('fma_pct', 0):.1f} | {d.get('warps_pct', 0):.1f} | {d.get('regs', 0):.0f} | "
                f"{d.get('grid', 0):.0f}×{d.get('block', 0):.0f} | {d.get('inst', 0):,.0f} | "
                f"{', '.join(d['stalls'])} |")
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    tp = os.path.join(os.path.dirname(a.out) or ".", "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt.setdefault(a.workload, {}).update(
        {k: sum(v) / len(v) for k, v in traffic.items()})
    json.dump(allt, open(tp, "w"), indent=1, sort_keys=True)
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
