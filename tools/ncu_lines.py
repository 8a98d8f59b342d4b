"""Join ncu per-SASS stall samples with CUDA source lines (nvdisasm -g of the
same build) and print the hottest source lines of a kernel.

    python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-name> [lib.so]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, kre, mangled = sys.argv[1:4]
    lib = sys.argv[4] if len(sys.argv) > 4 else "paper_2002_02885_b200/libpk_b200.so"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    data, hdr, k = [], None, 0
    for r in rows:
        if r and r[0] == "Kernel Name":
            k += 1
            if k > 1:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr:
            data.append(r)
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=td,
                       capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True,
                             text=True).stdout.splitlines()
    # walk the target function: track current source line per instruction
    in_fn, cur, lines = False, "?", []
    for ln in dis:
        if re.match(r"^\s*\.text\.", ln) or ln.startswith(".section"):
            in_fn = mangled in ln
            continue
        if not in_fn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
            lines.append(cur)
    agg = collections.Counter()
    why = collections.defaultdict(collections.Counter)
    stall_cols = [(j, h[6:]) for j, h in enumerate(hdr)
                  if h.startswith("stall_") and "Not Issued" not in h]
    iE = hdr.index("Instructions Executed")
    execd = collections.Counter()
    tot = 0
    for i, r in enumerate(data):
        s = int(r[iS])
        tot += s
        src = lines[i] if i < len(lines) else "?"
        agg[src] += s
        execd[src] += int(float(r[iE] or 0))
        for j, name in stall_cols:
            v = r[j]
            if v and float(v) > 0:
                why[src][name] += float(v)
    print(f"{len(data)} SASS rows, {len(lines)} disassembled, {tot} samples")
    if len(data) != len(lines):
        print("WARNING: the report and the library's SASS differ (the .ncu-rep was captured "
              "with another build): source lines below are not reliable")
    for src, s in agg.most_common(int(os.environ.get("TOP", "30"))):
        top = ", ".join(f"{n} {int(v)}" for n, v in why[src].most_common(3))
        print(f"{s:5d} {100 * s / tot:5.1f}%  {src:24s} inst {execd[src]:9d}  [{top}]")


if __name__ == "__main__":
    main()
