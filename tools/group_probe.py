"""Schedules of one ResNet-18 b256 step (packs + convs) timed as CUDA graphs: packs
alone, per-layer convs, one grouped conv, and their combinations on one stream.
Usage: python tools/group_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

A, W, B = 2, 1, 256
dev = torch.device("cuda")
stream = torch.cuda.Stream()
runs = []
for li in inputs.BASELINE_LAYERS:
    L = inputs.TABLE1[li]
    g = inputs.gen(li)
    act = inputs.codes((B, L.h, L.w, L.ic), A, g).to(dev)
    wt = inputs.codes((L.oc * L.k * L.k, L.ic), W, g).to(dev)
    packed = bs.bitpack(act, A)
    w_tc = bs.conv2d_tc_prepare_weights(bs.bitpack(wt, W), W, bs.BIPOLAR, L.oc, L.k, L.k, L.ic)
    oh = bs.conv_out_extent(L.h, L.k, L.s, L.pad)
    out = torch.empty((B, oh, oh, L.oc), dtype=torch.int32, device=dev)
    item = dict(act_packed=packed, w_tc=w_tc, out=out, n=B, h=L.h, w=L.w, c=L.ic, oc=L.oc, kh=L.k, kw=L.k,
                stride=L.s, pad=L.pad, w_enc=bs.BIPOLAR)
    runs.append((L, act, packed, item))


def packs(s):
    for L, act, packed, item in runs:
        bs.bitpack(act, A, out=packed, stream=s)


def packgroup(s):
    bs.bitpack_group([r[1] for r in runs], A, outs=[r[2] for r in runs], stream=s)


def convs(s):
    for L, act, packed, it in runs:
        bs.bitserial_conv2d_nhwc_tc_prepared(it["act_packed"], A, it["w_tc"], W, B, L.h, L.w, L.ic, L.oc, L.k, L.k,
                                             L.s, L.pad, out=it["out"], stream=s, w_enc=bs.BIPOLAR)


def group(s, sel=None):
    its = [r[3] for i, r in enumerate(runs) if sel is None or i in sel]
    bs.bitserial_conv2d_nhwc_tc_group(its, A, W, stream=s)


def interleaved(s):
    for L, act, packed, it in runs:
        bs.bitpack(act, A, out=packed, stream=s)
        bs.bitserial_conv2d_nhwc_tc_prepared(it["act_packed"], A, it["w_tc"], W, B, L.h, L.w, L.ic, L.oc, L.k, L.k,
                                             L.s, L.pad, out=it["out"], stream=s, w_enc=bs.BIPOLAR)


def t(fn, reps=10, trials=7):
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        fn(stream)
        stream.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for _ in range(reps):
                fn(stream)
        graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(trials):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            graph.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / reps * 1e3)
    return round(sorted(ts)[len(ts) // 2], 1)


res = {
    "packs": t(packs),
    "convs_per_layer": t(convs),
    "group_all": t(group),
    "group_no_L2": t(lambda s: group(s, set(range(1, 10)))),
    "packs+convs_serial": t(lambda s: (packs(s), convs(s))),
    "packs+group_serial": t(lambda s: (packs(s), group(s))),
    "interleaved_pack_conv": t(interleaved),
    "groups_5_5": t(lambda s: (group(s, set(range(5))), group(s, set(range(5, 10))))),
    "packgroup": t(packgroup),
    "packgroup+group_serial": t(lambda s: (packgroup(s), group(s))),
}
print(json.dumps(res))
