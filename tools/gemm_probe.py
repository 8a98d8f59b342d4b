"""Probe: TFLOP/s of one grouped conv GEMM launch (FPROP / DGRAD / WGRAD) built
through pk_cnn_prog for synthetic tensors.
    python tools/gemm_probe.py  (prints a table of shapes x N tiles)"""
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2002_02885_b200 import _lib, cnn  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()


def probe(mode, n, h, w, c, k, r, stride, K=4, nt=None, reps=20):
    pad = r // 2
    p = (h + 2 * pad - r) // stride + 1
    q = (w + 2 * pad - r) // stride + 1
    kpad = cnn.rup(r * r * c, 64)
    kpadt = cnn.rup(r * r * k, 64)
    structs, keep = [], []
    for _ in range(K):
        x = torch.randn(n * h * w, c, device=dev).to(torch.bfloat16)
        y = torch.randn(n * p * q, k, device=dev).to(torch.bfloat16)
        wt = torch.randn(k, kpad, device=dev).to(torch.bfloat16)
        wtt = torch.randn(c, kpadt, device=dev).to(torch.bfloat16)
        cs = _lib.CnnConv()
        cs.n, cs.h, cs.w, cs.c, cs.k, cs.r, cs.s = n, h, w, c, k, r, r
        cs.stride, cs.pad, cs.p, cs.q = stride, pad, p, q
        cs.ldx, cs.ldy = c, k
        if mode == "FPROP":
            cs.src, cs.wt, cs.dst, cs.ldo = x.data_ptr(), wt.data_ptr(), y.data_ptr(), k
            ntile = nt or cnn._pick_ntile(k)
            splits = 1
            keep += [x, y, wt]
        elif mode == "DGRAD":
            cs.src, cs.wt, cs.dst, cs.ldo = y.data_ptr(), wtt.data_ptr(), x.data_ptr(), c
            ntile = nt or cnn._pick_ntile(c)
            keep += [x, y, wtt]
        else:
            ntile, splits = cnn._wgrad_cfg(k, r * r * c, n * p * q)
            ntile = nt or ntile
            part = torch.empty(splits * k * kpad, device=dev)
            cs.src, cs.dy, cs.dst, cs.splits = x.data_ptr(), y.data_ptr(), part.data_ptr(), splits
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            cs.flag = flag.data_ptr()
            keep += [x, y, part, flag]
        structs.append(cs)
    kind = _lib.CNN["CONV_" + mode]
    prog = cnn.CnnProgram([(kind, (ntile, cnn._stages(ntile)), structs)], 0)
    st = torch.cuda.Stream()
    prog.run(st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, z in ev:
        a.record(st)
        prog.run(st.cuda_stream)
        z.record(st)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(z) for a, z in ev)
    M = n * p * q if mode != "DGRAD" else n * h * w
    fl = 2.0 * K * n * p * q * k * c * r * r
    print(f"{mode:5s} K={K} n{n} {h}x{w} c{c}->k{k} r{r} s{stride} NT={ntile:3d}: "
          f"{ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s", flush=True)


if __name__ != "__main__":
    pass
elif len(sys.argv) > 1 and sys.argv[1] == "one":  # one launch for ncu: one MODE n h w c k r halo cluster
    a = sys.argv[2:]
    _lib.set_plan_options(conv_halo=int(a[7]), conv_cluster=int(a[8]))
    probe(a[0], int(a[1]), int(a[2]), int(a[3]), int(a[4]), int(a[5]), int(a[6]), 1, reps=3)
elif len(sys.argv) > 1 and sys.argv[1] == "n64":  # N = 64 layers: im2col / pair MMA / halo
    for hl, cl in ((0, 0), (0, 1), (0, 2), (1, 1)):
        _lib.set_plan_options(conv_halo=hl, conv_cluster=cl)
        print("conv_halo", hl, "conv_cluster", cl)
        for mode in ("FPROP", "DGRAD"):
            probe(mode, 32, 56, 56, 64, 64, 3, 1)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "halo":  # conv_halo A/B (cluster off / on)
    for hl, cl in ((0, 1), (1, 1)):
        _lib.set_plan_options(conv_halo=hl, conv_cluster=cl)
        print("conv_halo", hl, "conv_cluster", cl)
        for mode in ("FPROP", "DGRAD"):
            probe(mode, 32, 56, 56, 64, 64, 3, 1)
            probe(mode, 32, 28, 28, 128, 128, 3, 1)
            probe(mode, 32, 14, 14, 256, 256, 3, 1)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "ab":  # conv_cluster A/B on FPROP / DGRAD
    for cl in [int(a) for a in sys.argv[2:]] or (0, 1, 2):
        _lib.set_plan_options(conv_cluster=cl)
        print("conv_cluster", cl)
        for mode in ("FPROP", "DGRAD"):
            probe(mode, 32, 56, 56, 64, 64, 3, 1)
            probe(mode, 32, 28, 28, 128, 128, 3, 1)
            probe(mode, 32, 14, 14, 256, 256, 3, 1)
            probe(mode, 32, 7, 7, 512, 512, 3, 1)
            probe(mode, 32, 56, 56, 256, 256, 1, 1)
    sys.exit(0)
if __name__ == "__main__" and (len(sys.argv) == 1):
  for mode in ("FPROP", "DGRAD", "WGRAD"):
    probe(mode, 32, 56, 56, 64, 64, 3, 1)
    probe(mode, 32, 28, 28, 128, 128, 3, 1)
    probe(mode, 32, 14, 14, 256, 256, 3, 1)
    probe(mode, 32, 7, 7, 512, 512, 3, 1)
    probe(mode, 32, 56, 56, 256, 256, 1, 1)   # a plain GEMM (1x1): M=100352, N=K=256
    probe(mode, 32, 56, 56, 256, 256, 1, 1, K=1)
  for nt in (64, 128, 256):
    probe("FPROP", 32, 14, 14, 256, 256, 3, 1, nt=nt)
    probe("FPROP", 32, 56, 56, 256, 256, 1, 1, nt=nt)
