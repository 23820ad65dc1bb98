"""Time the conv kernel of each BASELINE layer (batch 256 by default) for the library
selected by BITSERIAL_LIB (default: in-tree).  Each layer's launch is captured R times
back to back in a CUDA graph and timed with events around the replay (no host launch
overhead in the number); per-launch time = graph time / R, median over trials.
Usage: python tools/layer_sweep.py [--batch 256] [--a 2 --w 1] [--unipolar] [--tc] [--fused]"""
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
ap.add_argument("--reps", type=int, default=20, help="launches per graph")
ap.add_argument("--trials", type=int, default=5)
ap.add_argument("--layers", default=",".join(map(str, inputs.BASELINE_LAYERS)))
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--tc", action="store_true", help="tensor-core path on prepared weights")
ap.add_argument("--fused", action="store_true", help="include activation packing (the *_i8 entry)")
ap.add_argument("--raw", action="store_true",
                help="tensor cores on the PACKED weights (bs_bitserial_conv2d_nhwc, BS_ALGO_TC: weights expanded "
                     "in the kernel)")
ap.add_argument("--group", action="store_true",
                help="tensor-core path through bs_bitserial_conv2d_nhwc_tc_group: each layer as a group of one, "
                     "then all layers in one group")
ap.add_argument("--tile-n", type=int, default=0, help="BS_TUNE_TC_TILE_N (0 = library choice)")
args = ap.parse_args()
dev = torch.device("cuda")
if args.tile_n:
    bs.set_tuning(bs.TUNE_TC_TILE_N, args.tile_n)
enc = bs.UNIPOLAR if args.unipolar else bs.BIPOLAR
res = {}
tot_ops, tot_ms = 0, 0.0
stream = torch.cuda.Stream()
items = []


def time_graph(run):
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        run(stream)
        run(stream)
        stream.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for _ in range(args.reps):
                run(stream)
    graph.replay()
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(stream):  # replay() launches on the current stream: time that one
        for _ in range(args.trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / args.reps)
    del graph
    return sorted(ts)[len(ts) // 2]


for li in map(int, args.layers.split(",")):
    L = inputs.TABLE1[li]
    g = inputs.gen(li)
    act = inputs.codes((args.batch, L.h, L.w, L.ic), args.a, g).to(dev)
    wt = inputs.codes((L.oc * L.k * L.k, L.ic), args.w, g).to(dev)
    ap_ = bs.bitpack(act, args.a)
    wp = bs.bitpack(wt, args.w)
    oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
    out = torch.empty((args.batch, oh, oh, L.oc), dtype=torch.int32, device=dev)
    ws = torch.empty(max(16, bs.conv2d_workspace_bytes(args.batch, L.h, L.w, L.ic, args.a)), dtype=torch.uint8,
                     device=dev)
    w_tc = bs.conv2d_tc_prepare_weights(wp, args.w, enc, L.oc, L.k, L.k, L.ic) if args.tc else None
    if args.raw:
        run = lambda s: bs.bitserial_conv2d_nhwc(ap_, args.a, wp, args.w, enc, args.batch, L.h, L.w, L.ic, L.oc,  # noqa
                                                 L.k, L.k, L.s, L.pad, out=out, algo=bs.ALGO_TC, stream=s)
    elif args.group:
        item = dict(act_packed=ap_, w_tc=w_tc, out=out, n=args.batch, h=L.h, w=L.w, c=L.ic, oc=L.oc, kh=L.k, kw=L.k,
                    stride=L.s, pad=L.pad, w_enc=enc)
        items.append(item)
        run = lambda s, it=item: bs.bitserial_conv2d_nhwc_tc_group([it], args.a, args.w, stream=s)  # noqa
    elif args.tc and args.fused:
        run = lambda s: bs.bitserial_conv2d_nhwc_tc_i8(act, args.a, w_tc, args.w, L.oc, L.k, L.k, L.s, L.pad,  # noqa
                                                       out=out, workspace=ws, stream=s)
    elif args.tc:
        run = lambda s: bs.bitserial_conv2d_nhwc_tc_prepared(ap_, args.a, w_tc, args.w, args.batch, L.h, L.w,  # noqa
                                                             L.ic, L.oc, L.k, L.k, L.s, L.pad, out=out, stream=s)
    elif args.fused:
        run = lambda s: bs.bitserial_conv2d_nhwc_i8(act, args.a, wp, args.w, enc, L.oc, L.k, L.k, L.s, L.pad,  # noqa
                                                    out=out, workspace=ws, stream=s)
    else:
        run = lambda s: bs.bitserial_conv2d_nhwc(ap_, args.a, wp, args.w, enc, args.batch, L.h, L.w, L.ic, L.oc,  # noqa
                                                 L.k, L.k, L.s, L.pad, out=out, algo=args.algo, stream=s)
    ms = time_graph(run)
    ops = 2 * args.batch * oh * oh * L.oc * L.k * L.k * L.ic * args.a * args.w
    out_gb = out.numel() * 4 / 1e9
    res[li] = {"us": round(ms * 1e3, 2), "tops": round(ops / ms / 1e9, 1), "out_gbs": round(out_gb / ms * 1e3, 1)}
    tot_ops += ops
    tot_ms += ms
extra = {}
if args.group:
    extra["all_in_one_group_us"] = round(1e3 * time_graph(lambda s: bs.bitserial_conv2d_nhwc_tc_group(
        items, args.a, args.w, stream=s)), 2)
print(json.dumps({"lib": bs.library_path(), "tc": args.tc, "fused": args.fused, "a": args.a, "w": args.w,
                  "batch": args.batch, "bn": os.environ.get("BS_TC_BN"), "layers": res,
                  "total_us": round(tot_ms * 1e3, 1), "total_tops": round(tot_ops / tot_ms / 1e9, 1), **extra}))
