"""CPU tests of the conv pack path: the oracle's manual backward pinned against
torch autograd in float64, planner / oracle agreement on layer numbering and
init draws, every ctypes mirror of a pk_cnn_* struct checked against the C
header by compiling a probe with gcc, and the host planner's launch grouping
(no GPU needed: programs are only described, never created)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import cnn64 as O
from paper_2002_02885_b200 import _lib, cnn, packing

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMS = [("lenet5", 32, 1.0), ("mobilenetv2", 32, 0.5), ("resnet18", 32, 1.0),
        ("densenet121", 32, 1.0)]


def _autograd(spec, params, x, y):
    """torch autograd over the same net (fp64, training-mode BN)."""
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in params.items()}
    vals = {"input": x}
    pieces = {}   # concat buffer -> [(ch0, tensor)] written so far (DenseNet)

    def get(name):
        if name in spec.views:
            base, ch0, c = spec.views[name]
            parts = sorted(pieces[base], key=lambda t: t[0])
            return torch.cat([t for _, t in parts], dim=1)[:, ch0:ch0 + c]
        if name in pieces:
            return torch.cat([t for _, t in sorted(pieces[name], key=lambda t: t[0])], dim=1)
        return vals[name]

    def put(name, t):
        if name in spec.views:
            base, ch0, _ = spec.views[name]
            pieces.setdefault(base, []).append((ch0, t))
        else:
            vals[name] = t

    for L in spec.layers:
        n, xin = L["name"], get(L["x"])
        if L["kind"] == "conv":
            yv = F.conv2d(xin, P[n + "/W"].permute(0, 3, 1, 2), stride=L["stride"],
                          padding=L["pad"])
            if L["bias"]:
                yv = yv + P[n + "/b"].view(1, -1, 1, 1)
            put(L["y"], O._act(yv, L["act"]))
        elif L["kind"] == "bn":
            m = xin.mean(dim=(0, 2, 3))
            v = xin.var(dim=(0, 2, 3), unbiased=False)
            yv = ((xin - m.view(1, -1, 1, 1)) / torch.sqrt(v.view(1, -1, 1, 1) + O.BN_EPS)
                  * P[n + "/gamma"].view(1, -1, 1, 1) + P[n + "/beta"].view(1, -1, 1, 1))
            if L["res"]:
                yv = yv + get(L["res"])
            put(L["y"], O._act(yv, L["act"]))
        elif L["kind"] == "dw":
            vals[L["y"]] = F.conv2d(xin, P[n + "/W"].permute(2, 0, 1).unsqueeze(1),
                                    stride=L["stride"], padding=L["pad"], groups=L["c"])
        elif L["kind"] == "maxpool":
            put(L["y"], F.max_pool2d(xin, L["r"], L["stride"], L["pad"]))
        elif L["kind"] == "avgpool":
            put(L["y"], F.avg_pool2d(xin, L["r"], L["stride"], L["pad"]))
    loss = F.cross_entropy(get(spec.logits).reshape(x.shape[0], -1), y)
    loss.backward()
    return float(loss.detach()), {k: v.grad.numpy() for k, v in P.items()}


@pytest.mark.parametrize("fam,img,w", FAMS)
def test_oracle_backward_equals_autograd(fam, img, w):
    spec = O.Spec(fam, 10, (3, img, img), w)
    p = spec.init("m0", 0)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(6, 3, img, img, generator=g, dtype=torch.float64)
    y = torch.tensor([0, 1, 2, 3, 4, 5])
    l1, g1, _ = O.forward_backward(spec, p, x, y, mirror=False)
    l2, g2 = _autograd(spec, p, x, y)
    assert abs(l1 - l2) < 1e-12
    total = np.sqrt(sum(np.sum(v * v) for v in g2.values()))
    for k in g2:
        # elementwise to fp64 round-off of the whole gradient (analytically-zero
        # β gradients before a following BN are pure round-off on both sides)
        assert np.max(np.abs(g1[k] - g2[k])) <= 1e-10 * total, k


@pytest.mark.parametrize("fam,img,w", FAMS + [("resnet18", 224, 1.0)])
def test_planner_and_oracle_agree(fam, img, w):
    arch = cnn.ConvArch(fam, 10 if img == 32 else 1000, (3, img, img), w)
    net = cnn.build_net(arch)
    spec = O.Spec(fam, arch.classes, arch.image, w)
    assert spec.param_names() == [p.name for p in net.params]
    pi = cnn.init_parameters(net, "mX", 7)
    po = spec.init("mX", 7)
    for n in po:
        np.testing.assert_array_equal(pi["mX/" + n], po[n])
    for p in net.params:
        a = pi["mX/" + p.name]
        np.testing.assert_array_equal(cnn.from_dev_layout(p, cnn.to_dev_layout(p, a)),
                                      a.astype(np.float32).astype(np.float64))


def test_param_counts_match_torchvision_topologies():
    assert cnn.build_net(cnn.ConvArch("lenet5")).param_count == 62006
    assert cnn.build_net(cnn.ConvArch("densenet121", 1000, (3, 224, 224))).param_count == 7978856
    assert cnn.build_net(cnn.ConvArch("resnet18", 1000, (3, 224, 224))).param_count == 11689512
    # torchvision mobilenet_v2(width_mult=0.5, num_classes=10)
    assert cnn.build_net(cnn.ConvArch("mobilenetv2", 10, (3, 32, 32), 0.5)).param_count == 700490


def test_bf16_round_is_rne():
    a = np.array([1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -9, -2.5, 3.0e38, 1e-40], dtype=np.float32)
    want = torch.from_numpy(a).bfloat16().float().numpy().astype(np.float64)
    np.testing.assert_array_equal(cnn.bf16_round(a), want)


_PROBE = r'''
#include <stdio.h>
#include <stddef.h>
#include "packtrain_b200.h"
#define S(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  S(pk_cnn_conv) S(pk_cnn_bn) S(pk_cnn_dw) S(pk_cnn_pool) S(pk_cnn_head) S(pk_cnn_bias)
  S(pk_cnn_reduce) S(pk_cnn_opt_seg) S(pk_cnn_tpose) S(pk_cnn_commit) S(pk_cnn_op)
  S(pk_cnn_gather)
  O(pk_cnn_conv, n) O(pk_cnn_conv, nseg) O(pk_cnn_bn, rows) O(pk_cnn_bn, eps)
  O(pk_cnn_opt_seg, len) O(pk_cnn_opt_seg, wd) O(pk_cnn_head, ldl) O(pk_cnn_op, probs)
  printf("PK_CNN_NUM_KINDS %d\n", PK_CNN_NUM_KINDS);
  return 0;
}
'''

_PY = {"pk_cnn_conv": _lib.CnnConv, "pk_cnn_bn": _lib.CnnBn, "pk_cnn_dw": _lib.CnnDw,
       "pk_cnn_pool": _lib.CnnPool, "pk_cnn_head": _lib.CnnHead, "pk_cnn_bias": _lib.CnnBias,
       "pk_cnn_reduce": _lib.CnnReduce, "pk_cnn_opt_seg": _lib.CnnOptSeg,
       "pk_cnn_tpose": _lib.CnnTpose, "pk_cnn_commit": _lib.CnnCommit, "pk_cnn_op": _lib.CnnOp,
       "pk_cnn_gather": _lib.CnnGather}


def test_ctypes_structs_match_c_header(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(_PROBE)
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o",
                    str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, T in _PY.items():
        assert int(got[cname]) == ctypes.sizeof(T), cname
    for key, val in got.items():
        if "." in key:
            cname, field = key.split(".")
            assert getattr(_PY[cname], field).offset == int(val), key
    assert int(got["PK_CNN_NUM_KINDS"]) == len(_lib.CNN_KINDS)


def test_conv_handles_through_reference_api():
    arch = cnn.ConvArch("lenet5")
    hs = [packing.make_handle(f"m{i}", arch, "adam", 0.01, 16, 5, "train", 0) for i in range(2)]
    packed = packing.dedup_inputs(packing.pack_models(hs))
    assert packed.share_inputs and packed.driver_batch == 16
    assert [len(g) for g in packed.input_groups()] == [2]
    assert sorted(hs[0].params) == sorted(f"m0/{p.name}" for p in hs[0].net.params)
    with pytest.raises(packing.PackError):
        packing.pack_models([hs[0], packing.make_handle(
            "mlp", packing.MLPArch(3072, (16,), 10), "sgd", 0.1, 16, 5, "train", 0)])
