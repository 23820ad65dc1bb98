"""Time the conv kernel of each BASELINE layer (batch 256 by default) for the library
selected by BITSERIAL_LIB (default: in-tree).  Events around each launch, median of
reps.  Usage: python tools/layer_sweep.py [--batch 256] [--a 2 --w 1] [--unipolar]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--a", type=int, default=2)
ap.add_argument("--w", type=int, default=1)
ap.add_argument("--unipolar", action="store_true")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--layers", default=",".join(map(str, inputs.BASELINE_LAYERS)))
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--tc", action="store_true", help="tensor-core path (bs_bitserial_conv2d_nhwc_tc)")
args = ap.parse_args()
dev = torch.device("cuda")
enc = bs.UNIPOLAR if args.unipolar else bs.BIPOLAR
res = {}
tot_ops, tot_ms = 0, 0.0
for li in map(int, args.layers.split(",")):
    L = inputs.TABLE1[li]
    g = inputs.gen(li)
    act = inputs.codes((args.batch, L.h, L.w, L.ic), args.a, g).to(dev)
    wt = inputs.codes((L.oc * L.k * L.k, L.ic), args.w, g).to(dev)
    ap_ = bs.bitpack(act, args.a)
    wp = bs.bitpack(wt, args.w)
    out = torch.empty((args.batch, bs.conv_out_extent(L.h, L.k, L.s, L.pad), bs.conv_out_extent(L.w, L.k, L.s, L.pad),
                       L.oc), dtype=torch.int32, device=dev)
    ws = torch.empty(max(16, bs.conv2d_tc_workspace_bytes(L.oc, L.k, L.k, L.ic, args.w)), dtype=torch.uint8, device=dev)
    if args.tc:
        run = lambda: bs.bitserial_conv2d_nhwc_tc(ap_, args.a, wp, args.w, enc, args.batch, L.h, L.w, L.ic, L.oc,  # noqa
                                                  L.k, L.k, L.s, L.pad, out=out, workspace=ws)
    else:
        run = lambda: bs.bitserial_conv2d_nhwc(ap_, args.a, wp, args.w, enc, args.batch, L.h, L.w, L.ic, L.oc, L.k,  # noqa
                                               L.k, L.s, L.pad, out=out, algo=args.algo)
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
    ops = 2 * args.batch * oh * oh * L.oc * L.k * L.k * L.ic * args.a * args.w
    res[li] = {"ms": ms, "tops": ops / ms / 1e9}
    tot_ops += ops
    tot_ms += ms
print(json.dumps({"lib": bs.library_path(), "tc": args.tc, "a": args.a, "w": args.w, "layers": res, "total_ms": tot_ms,
                  "total_tops": tot_ops / tot_ms / 1e9}))
