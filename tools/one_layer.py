"""Run one ResNet layer's tensor-core conv (prepared weights, batch 256 A2W1 bipolar) a few
times: a small target for ncu captures.  Usage: python tools/one_layer.py LAYER [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

li = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L = inputs.TABLE1[li]
dev = torch.device("cuda")
g = inputs.gen(li)
act = inputs.codes((256, L.h, L.w, L.ic), 2, g).to(dev)
wt = inputs.codes((L.oc * L.k * L.k, L.ic), 1, g).to(dev)
ap_ = bs.bitpack(act, 2)
w_tc = bs.conv2d_tc_prepare_weights(bs.bitpack(wt, 1), 1, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
for _ in range(reps):
    bs.bitserial_conv2d_nhwc_tc_prepared(ap_, 2, w_tc, 1, 256, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad)
torch.cuda.synchronize()
print("ok")
