"""Per-step DRAM traffic per conv kernel kind from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(cache control none, one un-graphed step, tools/cnn_profile_step.py), merged
into profiles/ncu_traffic.json as {workload: {KIND: bytes per step}} (bench.py
reports it as roofline.traffic next to the algorithmic bytes).
    python tools/traffic_summary.py gpurun_out/<tag>/traffic_config1.csv config1"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = {"k_bn_stats": "BN_STATS", "k_bn_apply": "BN_APPLY", "k_bn_bwd_reduce": "BN_BWD_REDUCE",
        "k_bn_bwd_apply": "BN_BWD_APPLY", "k_dw_fprop": "DW_FPROP", "k_dw_dgrad": "DW_DGRAD",
        "k_dw_wgrad": "DW_WGRAD", "k_maxpool_fwd": "MAXPOOL_FWD", "k_maxpool_bwd": "MAXPOOL_BWD",
        "k_avgpool_fwd": "AVGPOOL_FWD", "k_avgpool_bwd": "AVGPOOL_BWD", "k_opt": "OPT",
        "k_conv_gemm<0>": "CONV_FPROP", "k_conv_gemm_p<0>": "CONV_FPROP",
        "k_conv_gemm<1>": "CONV_DGRAD", "k_conv_gemm_p<1>": "CONV_DGRAD",
        "k_conv_gemm<2>": "CONV_WGRAD", "k_conv_gemm_p<2>": "CONV_WGRAD",
        "k_split_reduce": "SPLIT_REDUCE", "k_publish_t": "PUBLISH_T", "k_xent": "XENT",
        "k_gather": "GATHER", "k_commit": "COMMIT", "k_im2col": "IM2COL"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, workload):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ni, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit", "ID"))
    per = collections.OrderedDict()   # launch id -> {kind, metrics}
    for r in rows[hi + 1:]:
        if len(r) <= vi or "at::" in r[ki]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        base = name.split("<")[0]
        base = base[:-2] if base.endswith("_t") else base  # specialised kernels (k_*_t<...>)
        kind = KIND.get(name) or KIND.get(base) or (
            {"k_conv_gemm_pc": "CONV", "k_conv_gemm_p2": "CONV", "k_conv_gemm_halo": "CONV",
             "k_conv_gemm_halo_res": "CONV"}.get(base, name))
        if kind == "CONV":
            kind = ("CONV_FPROP", "CONV_DGRAD", "CONV_WGRAD")[int(name.split("<")[1][0])]
        d = per.setdefault(r[ii], {"kind": kind})
        d[r[ni]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    launches = list(per.values())
    starts = [i for i, d in enumerate(launches) if d["kind"] == "GATHER"]
    step = launches[starts[-1]:] if starts else launches
    tot = collections.defaultdict(float)
    for d in step:
        tot[d["kind"]] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt[workload] = {k: round(v) for k, v in tot.items()}
    json.dump(allt, open(tp, "w"), indent=1, sort_keys=True)
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k:14s} {v / 1e6:10.1f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
