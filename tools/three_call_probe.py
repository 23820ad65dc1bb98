"""Time BASELINE configs[3] (ten ResNet-18 layers, batch 256, A2W1 bipolar) through the
north_star's three calls only (bs_bitpack of each layer's activations + bs_bitserial_conv2d_nhwc
on packed weights, AUTO -> tensor cores), eagerly and captured in one CUDA graph, beside the
per-layer device times of the same launches (tools only; parity is tests/test_parity_gpu.py).

    python tools/three_call_probe.py [--steps 20]
Prints one JSON object.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11066_b200 as bs  # noqa: E402
from paper_1810_11066_b200 import inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--tile-sweep", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
N = a.batch
runs = []
for li in inputs.BASELINE_LAYERS:
    L = inputs.TABLE1[li]
    act, wt = inputs.conv_operands(L, N, 2, 1, inputs.seed_for(4, 2, 1, "bipolar", li))
    act_d = act.to(dev)
    wp = bs.bitpack(wt.view(L.oc * L.k * L.k, L.ic).to(dev), 1)
    ap_ = bs.bitpack(act_d.view(-1, L.ic), 2)
    out = bs.bitserial_conv2d_nhwc(ap_, 2, wp, 1, bs.BIPOLAR, N, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad)
    runs.append(dict(li=li, L=L, act=act_d, wp=wp, ap=ap_, out=out))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def step():
    for r in runs:
        L = r["L"]
        bs.bitpack(r["act"].view(-1, L.ic), 2, out=r["ap"])
        bs.bitserial_conv2d_nhwc(r["ap"], 2, r["wp"], 1, bs.BIPOLAR, N, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad,
                                 out=r["out"])


def timed(fn, flush_l2=True):
    ts = []
    for i in range(3 + a.steps):
        if flush_l2:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


res = {"workload": "resnet18_layers2-12_b%d_a2w1_bipolar" % N, "calls": "bs_bitpack + bs_bitserial_conv2d_nhwc (AUTO)"}
res["eager_ms"] = timed(step)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
res["graph_ms"] = timed(g.replay)
per = []
for r in runs:
    L = r["L"]
    tp = timed(lambda: bs.bitpack(r["act"].view(-1, L.ic), 2, out=r["ap"]))
    tc = timed(lambda: bs.bitserial_conv2d_nhwc(r["ap"], 2, r["wp"], 1, bs.BIPOLAR, N, L.h, L.w, L.ic, L.oc, L.k,
                                                 L.k, L.s, L.pad, out=r["out"]))
    per.append({"layer": r["li"], "pack_us": tp * 1e3, "conv_us": tc * 1e3})
res["per_layer"] = per
if a.tile_sweep:  # the raw launch's tile width per layer: library choice vs forced 64 / 128
    sweep = []
    for r in runs:
        L = r["L"]
        row = {"layer": r["li"]}
        for bn in (0, 64, 128):
            bs.set_tuning(bs.TUNE_TC_TILE_N, bn)
            row["conv_us_bn%d" % bn] = 1e3 * timed(lambda: bs.bitserial_conv2d_nhwc(
                r["ap"], 2, r["wp"], 1, bs.BIPOLAR, N, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad, out=r["out"]))
        bs.set_tuning(bs.TUNE_TC_TILE_N, 0)
        sweep.append(row)
    res["tile_sweep"] = sweep
res["sum_per_layer_ms"] = sum(p["pack_us"] + p["conv_us"] for p in per) / 1e3
print(json.dumps(res))
