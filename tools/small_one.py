"""One small-path launch (bs_bitserial_conv2d_nhwc_i8_group) of ResNet layer LAYER at batch 1,
A2W1 bipolar, a few times: an ncu target.  Usage: python tools/small_one.py LAYER"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

li = int(sys.argv[1])
L = inputs.TABLE1[li]
act, wt = inputs.conv_operands(L, 1, 2, 1, li)
it = dict(act=act.cuda(), w_packed=bs.bitpack(wt.view(-1, L.ic).cuda(), 1), w_enc=bs.BIPOLAR, oc=L.oc, kh=L.k,
          kw=L.k, stride=L.s, pad=L.pad)
for _ in range(3):
    bs.bitserial_conv2d_nhwc_i8_group([it], 2, 1)
torch.cuda.synchronize()
print("ok")
