"""Per-role wait cycles of CTA 0 (BS_TC_PROFILE build: BITSERIAL_LIB=build/libbitserial_prof.so)
for single tensor-core conv launches of the given ResNet layers at batch 256.
Usage: BITSERIAL_LIB=build/libbitserial_prof.so python tools/prof_probe.py [--raw] 2 6 12
(--raw: the three-call boundary's launch, packed weight planes expanded in the kernel)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

dev = torch.device("cuda")
raw = "--raw" in sys.argv
for li in [int(x) for x in sys.argv[1:] if x != "--raw"]:
    L = inputs.TABLE1[li]
    g = inputs.gen(li)
    act = inputs.codes((256, L.h, L.w, L.ic), 2, g).to(dev)
    wt = inputs.codes((L.oc * L.k * L.k, L.ic), 1, g).to(dev)
    ap_ = bs.bitpack(act, 2)
    w_tc = bs.conv2d_tc_prepare_weights(bs.bitpack(wt, 1), 1, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
    wp = bs.bitpack(wt, 1)
    if raw:
        run = lambda: bs.bitserial_conv2d_nhwc(ap_, 2, wp, 1, bs.BIPOLAR, 256, L.h, L.w, L.ic, L.oc, L.k, L.k,  # noqa
                                               L.s, L.pad, algo=bs.ALGO_TC)
    else:
        run = lambda: bs.bitserial_conv2d_nhwc_tc_prepared(ap_, 2, w_tc, 1, 256, L.h, L.w, L.ic, L.oc, L.k,  # noqa
                                                           L.k, L.s, L.pad)
    run()
    torch.cuda.synchronize()
    print(f"=== layer {li} ===", flush=True)
    run()
    torch.cuda.synchronize()
    print(f"=== end {li} ===", flush=True)
