"""Run the window-path conv of ResNet-18 layers (A2W1 bipolar) a few times — a target for ncu
captures (tools only; no timing printed).

    python tools/tcw_one.py --layers 11 [--iters 3] [--group] [--batch 256]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tcw_probe import setup  # noqa: E402
import paper_1810_11066_b200 as bs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="11")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--group", action="store_true")
ap.add_argument("--batch", type=int, default=256)
a = ap.parse_args()
runs = setup(a.batch, 2, 1, [int(x) for x in a.layers.split(",")])
bs.digitpack_win_group([r["pk"] for r in runs], 2, outs=[r["aw"] for r in runs])
for _ in range(a.iters):
    if a.group:
        bs.bitserial_conv2d_nhwc_tcw_group([r["item"] for r in runs], 2, 1)
    else:
        for r in runs:
            bs.bitserial_conv2d_nhwc_tcw_group([r["item"]], 2, 1)
torch.cuda.synchronize()
print("ok")
