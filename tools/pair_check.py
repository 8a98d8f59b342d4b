"""Check: CTA-pair GEMM (plan conv_cluster=2) equals the one-CTA GEMM bit for bit
on FPROP / DGRAD problems (256 / 128-wide N tiles, odd M-tile counts)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2002_02885_b200 import _lib, cnn  # noqa: E402

dev = torch.device("cuda", 0)


def run(mode, n, h, w, c, k, r, cl):
    _lib.set_plan_options(conv_cluster=cl)
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
for args in (("FPROP", 8, 14, 14, 256, 256, 3), ("DGRAD", 8, 14, 14, 256, 256, 3),
             ("FPROP", 3, 7, 7, 512, 512, 3), ("FPROP", 4, 28, 28, 128, 128, 3),
             ("DGRAD", 4, 28, 28, 128, 128, 3), ("FPROP", 5, 9, 9, 256, 256, 1)):
    a = run(*args, 0)
    b = run(*args, 2)
    same = torch.equal(a, b)
    ok &= same
    print(args, "pair == one-CTA:", same, "max |diff|", float((a - b).abs().max()), flush=True)
print("ALL OK" if ok else "MISMATCH")
