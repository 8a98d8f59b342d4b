"""Check: a conv GEMM plan variant against the plain one-CTA TMA im2col GEMM on
FPROP / DGRAD problems.   python tools/pair_check.py [pair|halo]
  pair: plan conv_cluster=2 (CTA-pair MMA) must be bit-identical;
  halo: plan conv_halo=1 (halo tiles) bit-identical for C == 64, else within
        fp32 reordering (|Δ| <= 2^-7 |ref| + 1e-3 max|ref| on the bf16 outputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2002_02885_b200 import _lib, cnn  # noqa: E402

dev = torch.device("cuda", 0)


VARIANT = sys.argv[1] if len(sys.argv) > 1 else "pair"


def run(mode, n, h, w, c, k, r, on):
    if VARIANT == "pair":
        _lib.set_plan_options(conv_cluster=2 if on else 0, conv_halo=0)
    else:
        _lib.set_plan_options(conv_cluster=0, conv_halo=1 if on else 0)
    torch.manual_seed(0)
    pad = r // 2
    p, q = h, w
    kpad, kpadt = cnn.rup(r * r * c, 64), cnn.rup(r * r * k, 64)
    x = torch.randn(n * h * w, c, device=dev).to(torch.bfloat16)
    y = torch.randn(n * p * q, k, device=dev).to(torch.bfloat16)
    wt = torch.randn(k, kpad, device=dev).to(torch.bfloat16)
    wtt = torch.randn(c, kpadt, device=dev).to(torch.bfloat16)
    cs = _lib.CnnConv()
    cs.n, cs.h, cs.w, cs.c, cs.k, cs.r, cs.s = n, h, w, c, k, r, r
    cs.stride, cs.pad, cs.p, cs.q = 1, pad, p, q
    cs.ldx, cs.ldy = c, k
    if mode == "FPROP":
        out = torch.zeros(n * p * q, k, device=dev, dtype=torch.bfloat16)
        cs.src, cs.wt, cs.dst, cs.ldo = x.data_ptr(), wt.data_ptr(), out.data_ptr(), k
        nt = cnn._pick_ntile(k)
    else:
        out = torch.zeros(n * h * w, c, device=dev, dtype=torch.bfloat16)
        cs.src, cs.wt, cs.dst, cs.ldo = y.data_ptr(), wtt.data_ptr(), out.data_ptr(), c
        nt = cnn._pick_ntile(c)
    prog = cnn.CnnProgram([(_lib.CNN["CONV_" + mode], (nt, cnn._stages(nt)), [cs])], 0)
    st = torch.cuda.Stream()
    prog.run(st.cuda_stream)
    torch.cuda.synchronize()
    return out.float().cpu()


ok = True
cases = ((("FPROP", 8, 14, 14, 256, 256, 3), ("DGRAD", 8, 14, 14, 256, 256, 3),
          ("FPROP", 4, 56, 56, 64, 64, 3), ("DGRAD", 3, 28, 28, 64, 64, 3),
          ("FPROP", 3, 7, 7, 512, 512, 3), ("FPROP", 4, 28, 28, 128, 128, 3),
          ("DGRAD", 4, 28, 28, 128, 128, 3), ("FPROP", 5, 9, 9, 256, 256, 1))
         if VARIANT == "pair" else
         (("FPROP", 4, 56, 56, 64, 64, 3), ("DGRAD", 4, 56, 56, 64, 64, 3),
          ("FPROP", 3, 28, 28, 128, 128, 3), ("DGRAD", 3, 28, 28, 128, 128, 3),
          ("FPROP", 5, 14, 14, 256, 256, 3), ("DGRAD", 5, 14, 14, 256, 256, 3),
          ("FPROP", 2, 15, 17, 64, 96, 3), ("FPROP", 2, 14, 14, 64, 32, 3)))
for args in cases:
    a = run(*args, False)
    b = run(*args, True)
    same = torch.equal(a, b)
    d = float((a - b).abs().max())
    close = bool(((a - b).abs() <= 2 ** -7 * a.abs() + 1e-3 * a.abs().max()).all())
    good = same if (VARIANT == "pair" or args[4 if args[0] == "FPROP" else 5] == 64) else close
    ok &= good
    print(args, VARIANT, "identical:", same, "close:", close, "max |diff|", d, flush=True)
print("ALL OK" if ok else "MISMATCH")
