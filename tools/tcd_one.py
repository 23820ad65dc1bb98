"""Run the digit-path conv of ResNet-18 layers (batch 256, A2W1 bipolar) a few times — a
target for ncu captures (tools only; no timing printed).

    python tools/tcd_one.py --layers 5 [--iters 3] [--group]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tcd_probe import conv_setup  # noqa: E402
import paper_1810_11066_b200 as bs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="5")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--group", action="store_true", help="all listed layers in one grouped launch")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--gemm", type=int, default=0, help="M=N=K of a dense A2W1 product instead of conv layers")
ap.add_argument("--tile-n", type=int, default=0)
ap.add_argument("--asrc", type=int, default=0)
a = ap.parse_args()
bs.set_tuning(bs.TUNE_TCD_A_SRC, a.asrc)
if a.tile_n:
    bs.set_tuning(bs.TUNE_TC_TILE_N, a.tile_n)
if a.gemm:
    from paper_1810_11066_b200 import inputs
    g = inputs.gen(a.gemm)
    A = inputs.codes((a.gemm, a.gemm), 2, g).to("cuda")
    W = inputs.codes((a.gemm, a.gemm), 1, g).to("cuda")
    ad = bs.digitpack(A, 2)
    wd = bs.dense_tcd_prepare_weights(bs.bitpack(W, 1), 1, bs.BIPOLAR, a.gemm, a.gemm)
    for _ in range(a.iters):
        bs.bitserial_dense_tcd(ad, 2, wd, 1, a.gemm, a.gemm, a.gemm, w_enc=1)
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
layers = [int(x) for x in a.layers.split(",")]
runs = conv_setup(a.batch, 2, 1, layers)
bs.digitpack_group([r["act"] for r in runs], 2, outs=[r["ad"] for r in runs])
for _ in range(a.iters):
    if a.group:
        bs.bitserial_conv2d_nhwc_tcd_group([r["item"] for r in runs], 2, 1)
    else:
        for r in runs:
            bs.bitserial_conv2d_nhwc_tcd_group([r["item"]], 2, 1)
torch.cuda.synchronize()
print("ok")
