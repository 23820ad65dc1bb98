"""Time the one-launch small-problem path (bs_bitserial_conv2d_nhwc_i8_group) for the
batch-1 configs at each K split (cluster size), graph-replayed (per-launch us).
Usage: python tools/small_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

dev = torch.device("cuda")


def graph_us(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(s)
            g.replay()
            e1.record(s)
            s.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best


def items(layers):
    out = []
    for li in layers:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, 1, 2, 1, li)
        out.append(dict(act=act.to(dev), w_packed=bs.bitpack(wt.view(-1, L.ic).to(dev), 1), w_enc=bs.BIPOLAR,
                        oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad))
    return out


res = {}
for name, layers in (("conv1", (2,)), ("resnet1", inputs.BASELINE_LAYERS)):
    its = items(layers)
    for ks in (0, 1, 2, 4, 8):
        bs.set_tuning(bs.TUNE_SMALL_KSPLIT, ks)
        res[f"{name}_ks{ks}"] = round(graph_us(lambda: bs.bitserial_conv2d_nhwc_i8_group(its, 2, 1)), 2)
    bs.set_tuning(bs.TUNE_SMALL_KSPLIT, 0)
    for li, it in zip(layers, its):
        res[f"{name}_L{li}"] = round(graph_us(lambda it=it: bs.bitserial_conv2d_nhwc_i8_group([it], 2, 1)), 2)
empty = torch.empty(16, device=dev)
res["empty_kernel"] = round(graph_us(lambda: empty.zero_()), 2)
print(json.dumps(res))
