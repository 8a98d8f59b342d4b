"""The committed bench lines (profiles/r1ar, measured on a B200) keep bench.py's
JSON contract: whole-job value, e2e through the packing API with host copies
counted, roofline of the top phase against the measured peak, the CPU
reference timed beside it, clocks sampled under load, and the DRAM traffic of
the top kernel present in profiles/ncu_traffic.json (what bench.py reports as
`roofline.traffic`). CPU-only: reads JSON files, runs nothing."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = os.path.join(ROOT, "profiles", "r1ar")
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e")


def _line(name):
    with open(os.path.join(RUN, name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


@pytest.mark.parametrize("name", ["bench.json", "bench_k16.json", "bench_wide16.json"])
def test_own_arm_line(name):
    d = _line(name)
    for k in BASE_KEYS + ("roofline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["config"]["workload"] in ("config0", "k16", "wide16")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                              "sw_thermal_slowdown"}
    traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    kname = r["kernel"].split("[")[0]
    assert kname in traffic[d["config"]["workload"]]


def test_headline_cpu_baseline_is_the_reference():
    d = _line("bench.json")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] > 0
    assert d["config"]["workload"] == "config0"


def test_reference_arm_line():
    d = _line("bench_ref.json")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"],
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    own = _line("bench.json")
    assert (d["metric"], d["unit"], d["higher_is_better"]) == (
        own["metric"], own["unit"], own["higher_is_better"])
    assert d["config"]["workload"] == own["config"]["workload"]


def test_gpus_flag_launches_that_many_ranks():
    """`python bench.py --gpus 2` (no torchrun) must run 2 ranks, one per GPU:
    the launcher re-executes itself under torch.distributed.run (dry-run hook,
    no device work)."""
    import subprocess
    import sys
    env = dict(os.environ, PK_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)
